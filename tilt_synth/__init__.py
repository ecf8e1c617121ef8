"""Seeded synthetic inputs for the TILT hot path (shared by the oracle tests and the GPU path).

This module only *generates inputs*: canvases, boxes, initial transforms and the planted ground
truth. It holds none of the method's arithmetic (no warp/Jacobian, no projector, no LADMAP), so the
fp64 oracle (``oracle/``) and the CUDA path (``paper_1205_5351_b200``) stay independent.

The paper's datasets are not available, so these stand in for
them, with the shapes of BASELINE.json's configs and the paper's affine parameterisation
``A(theta, t) = R(theta) [[1, t], [0, 1]]`` (§6.2 "Range of Convergence").
Recipe:

* canvas 2m x 2n fp32, the box is the central m x n window;
* texture ``T = sum_k a_k b_k^T`` with a_k, b_k piecewise-constant vectors (segment lengths
  U{ceil(N/16)..ceil(N/6)} px, values U[0,1]) rescaled to [0,1], optionally blurred;
* canvas pixel x shows ``T(H_G^{-1}(x - c))`` (normalised frame of DESIGN.md reading R1),
  2x2 supersampled;
* corruption replaces exactly round(f * 4mn) canvas pixels by U[0,1] (reading Z23),
  then optional Gaussian noise.

Everything is drawn from ``numpy.random.default_rng([config_id, patch_index])`` so every rank can
generate its own shard without communication.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

AFFINE = 0
HOMOGRAPHY = 1


@dataclasses.dataclass(frozen=True)
class SynthConfig:
    """One BASELINE.json config (indices follow BASELINE.json ``configs`` order, 1-based)."""

    config_id: int
    batch: int
    m: int
    n: int
    kind: int
    rank_lo: int
    rank_hi: int
    theta_deg: float  # rotation drawn from U[-theta, theta]
    skew: float  # skew drawn from U[-skew, skew]
    persp_px: float  # h31, h32 drawn from U[-persp, persp] in pixel units (reading Z17)
    corrupt: float  # fraction of canvas pixels replaced by U[0, 1]
    noise: float = 0.0
    pyramid_levels: int = 1
    blur_px: float = 0.0

    @property
    def p(self) -> int:
        return 6 if self.kind == AFFINE else 8


CONFIGS = {
    # BASELINE.json configs[0]: 1 patch 32x32, affine, rank 2, rot U[-15,15] deg, skew U[-0.2,0.2], 5%.
    1: SynthConfig(1, 1, 32, 32, AFFINE, 2, 2, 15.0, 0.2, 0.0, 0.05),
    # configs[1]: 1024 x 50x50 homography, r in U{2..5}, rot +-30, skew +-0.3, persp +-1e-3, 10%.
    2: SynthConfig(2, 1024, 50, 50, HOMOGRAPHY, 2, 5, 30.0, 0.3, 1e-3, 0.10),
    # configs[2]: 4096 x 100x100 homography, 2-level pyramid, rank 3, rot +-30, 10%, noise 0.01.
    3: SynthConfig(3, 4096, 100, 100, HOMOGRAPHY, 3, 3, 30.0, 0.0, 0.0, 0.10, 0.01, 2),
    # configs[3]: 256 x 200x200 affine, r in U{2..8}, rot +-45, skew +-0.4, 20%.
    4: SynthConfig(4, 256, 200, 200, AFFINE, 2, 8, 45.0, 0.4, 0.0, 0.20),
    # configs[4]: 65536 x 50x50 as config 2 (sharded across GPUs).
    5: SynthConfig(5, 65536, 50, 50, HOMOGRAPHY, 2, 5, 30.0, 0.3, 1e-3, 0.10),
}


def _piecewise_constant(rng: np.random.Generator, length: int, seg_lo: int, seg_hi: int) -> np.ndarray:
    out = np.empty(length, dtype=np.float64)
    pos = 0
    while pos < length:
        seg = int(rng.integers(seg_lo, seg_hi + 1))
        out[pos:pos + seg] = rng.uniform(0.0, 1.0)
        pos += seg
    lo, hi = out.min(), out.max()
    return (out - lo) / (hi - lo) if hi > lo else out * 0.0


def _blur(vec: np.ndarray, sigma: float) -> np.ndarray:
    if sigma <= 0:
        return vec
    r = int(math.ceil(4 * sigma))
    k = np.exp(-0.5 * (np.arange(-r, r + 1) / sigma) ** 2)
    k /= k.sum()
    return np.convolve(np.pad(vec, r, mode="edge"), k, mode="valid")


def planted_transform(theta: float, skew: float, h31: float = 0.0, h32: float = 0.0) -> np.ndarray:
    """H_G = [[A, 0], [h31, h32, 1]], A = R(theta) [[1, skew], [0, 1]]."""
    c, s = math.cos(theta), math.sin(theta)
    a = np.array([[c, -s], [s, c]]) @ np.array([[1.0, skew], [0.0, 1.0]])
    h = np.eye(3)
    h[:2, :2] = a
    h[2, 0], h[2, 1] = h31, h32
    return h


def tau_from_h(h: np.ndarray, kind: int) -> np.ndarray:
    """Parameter order (h11, h12, h21, h22, h13, h23[, h31, h32]) (reading Z16)."""
    t = [h[0, 0], h[0, 1], h[1, 0], h[1, 1], h[0, 2], h[1, 2]]
    if kind == HOMOGRAPHY:
        t += [h[2, 0], h[2, 1]]
    return np.asarray(t, dtype=np.float64)


def identity_tau(kind: int) -> np.ndarray:
    return tau_from_h(np.eye(3), kind)


def render_texture(a: list, b: list, h_g: np.ndarray, m: int, n: int, box_xy: tuple,
                   canvas_hw: tuple, supersample: int = 2) -> np.ndarray:
    """Canvas pixel (X, Y) shows T(H_G^{-1}((X, Y) - c) / s) with T(u, v) = sum_k a_k(v) b_k(u)."""
    hc, wc = canvas_hw
    x0, y0 = box_xy
    s = max(m, n) / 2.0
    cx, cy = x0 + (n - 1) / 2.0, y0 + (m - 1) / 2.0
    offs = (np.arange(supersample) + 0.5) / supersample - 0.5
    ys = (np.arange(hc)[:, None] + offs[None, :]).reshape(-1)
    xs = (np.arange(wc)[:, None] + offs[None, :]).reshape(-1)
    gx, gy = np.meshgrid((xs - cx) / s, (ys - cy) / s)
    hinv = np.linalg.inv(h_g)
    den = hinv[2, 0] * gx + hinv[2, 1] * gy + hinv[2, 2]
    u = (hinv[0, 0] * gx + hinv[0, 1] * gy + hinv[0, 2]) / den
    v = (hinv[1, 0] * gx + hinv[1, 1] * gy + hinv[1, 2]) / den
    length = a[0].shape[0]
    iu = np.clip(np.floor(u * s + length / 2.0).astype(np.int64), 0, length - 1)
    iv = np.clip(np.floor(v * s + length / 2.0).astype(np.int64), 0, length - 1)
    tex = np.zeros_like(u)
    for ak, bk in zip(a, b):
        tex += ak[iv] * bk[iu]
    tex /= len(a)
    tex = tex.reshape(hc, supersample, wc, supersample).mean(axis=(1, 3))
    return tex


def gen_patch(cfg: SynthConfig, idx: int, *, planted: bool = True, blur_px: float | None = None,
              rank: int | None = None) -> dict:
    """Canvas + box + tau0 + ground truth for patch ``idx`` of ``cfg`` (seed [config_id, idx])."""
    rng = np.random.default_rng([cfg.config_id, idx])
    m, n = cfg.m, cfg.n
    big = max(m, n)
    r = int(rng.integers(cfg.rank_lo, cfg.rank_hi + 1)) if rank is None else rank
    theta = math.radians(rng.uniform(-cfg.theta_deg, cfg.theta_deg))
    skew = rng.uniform(-cfg.skew, cfg.skew) if cfg.skew > 0 else 0.0
    if cfg.kind == HOMOGRAPHY and cfg.persp_px > 0:
        p31, p32 = rng.uniform(-cfg.persp_px, cfg.persp_px, size=2)
    else:
        p31 = p32 = 0.0
    length = 8 * big
    seg_lo, seg_hi = math.ceil(big / 16), math.ceil(big / 6)
    blur = cfg.blur_px if blur_px is None else blur_px
    a = [_blur(_piecewise_constant(rng, length, seg_lo, seg_hi), blur) for _ in range(r)]
    b = [_blur(_piecewise_constant(rng, length, seg_lo, seg_hi), blur) for _ in range(r)]
    s = big / 2.0
    if not planted:
        theta, skew, p31, p32 = 0.0, 0.0, 0.0, 0.0
    h_g = planted_transform(theta, skew, p31 * s, p32 * s)
    hc, wc = 2 * m, 2 * n
    x0, y0 = n // 2, m // 2
    canvas = render_texture(a, b, h_g, m, n, (x0, y0), (hc, wc))
    npx = hc * wc
    k = int(round(cfg.corrupt * npx))
    if k > 0:
        sel = rng.choice(npx, size=k, replace=False)
        flat = canvas.reshape(-1)
        flat[sel] = rng.uniform(0.0, 1.0, size=k)
    if cfg.noise > 0:
        canvas = canvas + rng.normal(0.0, cfg.noise, size=canvas.shape)
    return {
        "canvas": canvas.astype(np.float32),
        "box": np.array([x0, y0, n, m], dtype=np.int32),
        "tau0": identity_tau(cfg.kind),
        "tau_g": tau_from_h(h_g, cfg.kind),
        "rank": r,
        "theta": theta,
        "skew": skew,
    }


def gen_batch(cfg: SynthConfig, start: int = 0, count: int | None = None, **kw) -> dict:
    """Patches [start, start+count) of ``cfg``: one canvas per patch (patch_image = arange)."""
    count = cfg.batch if count is None else count
    pats = [gen_patch(cfg, start + i, **kw) for i in range(count)]
    if count == 0:
        hc, wc = 2 * cfg.m, 2 * cfg.n
        return {"images": np.zeros((0, hc, wc), np.float32), "patch_image": np.zeros(0, np.int32),
                "boxes": np.zeros((0, 4), np.int32), "tau0": np.zeros((0, cfg.p)),
                "tau_g": np.zeros((0, cfg.p)), "rank": np.zeros(0, np.int32)}
    return {
        "images": np.stack([p["canvas"] for p in pats]),
        "patch_image": np.arange(count, dtype=np.int32),
        "boxes": np.stack([p["box"] for p in pats]),
        "tau0": np.stack([p["tau0"] for p in pats]),
        "tau_g": np.stack([p["tau_g"] for p in pats]),
        "rank": np.array([p["rank"] for p in pats], dtype=np.int32),
    }


def table1_instance(n: int, p: int, seed: int, m: int | None = None) -> dict:
    """Table 1's random inner-loop data (reading Z20).

    D ~ U[-1/2, 1/2]^{m x n} (unnormalised), J ~ N(0, 1)^{mn x p}, lambda = 1/sqrt(max(m, n)).
    J is returned as p planes of shape (m, n) (row-major pixel order, reading Z1).
    """
    m = n if m is None else m
    rng = np.random.default_rng([1001, n, p, seed])
    d = rng.uniform(-0.5, 0.5, size=(m, n))
    j = rng.normal(0.0, 1.0, size=(p, m, n))
    return {"D": d, "J": j, "lam": 1.0 / math.sqrt(max(m, n))}


def lowrank_sparse(m: int, n: int, rank: int, seed: int, frac: float = 0.05) -> np.ndarray:
    """A unit-norm low-rank + sparse + small-noise matrix (SVT / inner-loop parity inputs)."""
    rng = np.random.default_rng([1002, m, n, rank, seed])
    x = rng.normal(size=(m, rank)) @ rng.normal(size=(rank, n))
    k = int(round(frac * m * n))
    sel = rng.choice(m * n, size=k, replace=False)
    x.reshape(-1)[sel] += rng.normal(0, 3.0, size=k)
    x += 1e-3 * rng.normal(size=(m, n))
    return x / np.linalg.norm(x)


def checkerboard_case(theta: float, skew: float, m: int = 32, square_px: int = 8, supersample: int = 4) -> dict:
    """Fig. 2's range-of-convergence input: a standard 0/1 checker-board
    (squares of ``square_px`` window pixels) deformed by y = A(theta, t) x, A(theta, t) =
    R(theta) [[1, t], [0, 1]], on a 2m x 2m canvas with the central m x m window; no corruption.
    The checker-board is T(u, v) = (1 + s(u) s(v)) / 2 with s a +-1 square wave (rank 2)."""
    big = m
    length = 8 * big
    wave = np.where((np.arange(length) // square_px) % 2 == 0, 1.0, -1.0)
    ones = np.ones(length)
    h_g = planted_transform(theta, skew)
    x0 = y0 = m // 2
    canvas = render_texture([ones, wave], [ones, wave], h_g, m, m, (x0, y0), (2 * m, 2 * m), supersample)
    return {"canvas": canvas.astype(np.float32), "box": np.array([x0, y0, m, m], dtype=np.int32),
            "tau0": identity_tau(AFFINE), "tau_g": tau_from_h(h_g, AFFINE), "theta": theta, "skew": skew}


def convergence_grid(m: int = 32, square_px: int = 8) -> dict:
    """The Fig. 2 grid: theta in [0, pi/6] step pi/60, t in [0, 1] step 0.05."""
    thetas = [k * math.pi / 60 for k in range(11)]
    skews = [round(0.05 * k, 2) for k in range(21)]
    cases = [checkerboard_case(th, t, m, square_px) for th in thetas for t in skews]
    return {"thetas": thetas, "skews": skews,
            "images": np.stack([c["canvas"] for c in cases]),
            "patch_image": np.arange(len(cases), dtype=np.int32),
            "boxes": np.stack([c["box"] for c in cases]),
            "tau0": np.stack([c["tau0"] for c in cases]),
            "tau_g": np.stack([c["tau_g"] for c in cases])}



def corruption_case(idx: int, frac: float, m: int = 32, theta_deg: float = 10.0, rank: int = 3) -> dict:
    """Fig. 4's robustness input (synthetic stand-in for the missing
    low-rank-texture set): texture ``idx`` (seed [6, idx]: rank-``rank`` piecewise-constant, as the
    configs), rotated by ``theta_deg`` (the paper's 10 degrees), then exactly round(frac * 4 m^2)
    canvas pixels replaced by U[0, 1] (seed [6, idx, round(1000 frac)], reading Z23)."""
    rng = np.random.default_rng([6, idx])
    length = 8 * m
    seg_lo, seg_hi = math.ceil(m / 16), math.ceil(m / 6)
    a = [_piecewise_constant(rng, length, seg_lo, seg_hi) for _ in range(rank)]
    b = [_piecewise_constant(rng, length, seg_lo, seg_hi) for _ in range(rank)]
    h_g = planted_transform(math.radians(theta_deg), 0.0)
    x0 = y0 = m // 2
    canvas = render_texture(a, b, h_g, m, m, (x0, y0), (2 * m, 2 * m))
    npx = 4 * m * m
    k = int(round(frac * npx))
    if k > 0:
        r2 = np.random.default_rng([6, idx, int(round(1000 * frac))])
        sel = r2.choice(npx, size=k, replace=False)
        canvas.reshape(-1)[sel] = r2.uniform(0.0, 1.0, size=k)
    return {"canvas": canvas.astype(np.float32), "box": np.array([x0, y0, m, m], dtype=np.int32),
            "tau0": identity_tau(AFFINE), "tau_g": tau_from_h(h_g, AFFINE)}
