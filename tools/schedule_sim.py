"""Scheduling model of the persistent CTA-per-patch solve (tail-effect analysis).

Input: per-patch inner-iteration counts of the bench batch (tools/patch_costs.py). Model: 148 SMs
with up to 4 resident patches each; a patch advances at the measured per-CTA rate for its SM's
load (tools/prof_solve.py at 148/296/592 patches: 8.46k / 6.25k / ~4.8k / 3.77k iterations/s per
CTA at 1/2/3/4 CTAs per SM); a freed slot takes the next patch of the queue. Compares the queue
order of the kernel (patch index), longest-first (an oracle order), the perfectly packed bulk, and
a two-phase variant (iteration budget, then the suspended patches alone on an SM).
Usage: python tools/schedule_sim.py [costs.npz]"""
import sys

import numpy as np

path = sys.argv[1] if len(sys.argv) > 1 else "profiles/r01/schedule/bench_batch_costs.npz"
d = np.load(path)
W = d["inner"].astype(float)
RATES = {1: 8460.0, 2: 6250.0, 3: 4800.0, 4: 3770.0}
NSM, CAP = 148, 4


def simulate(work, order, cap=CAP, rates=RATES):
    queue = list(order)
    rem, sm_of, load, active, t = {}, {}, [0] * NSM, [], 0.0
    for s in [s for _ in range(cap) for s in range(NSM)]:
        if not queue:
            break
        p = queue.pop(0)
        rem[p], sm_of[p] = work[p], s
        load[s] += 1
        active.append(p)
    while active:
        dt = min(rem[p] / rates[load[sm_of[p]]] for p in active)
        for p in active:
            rem[p] -= dt * rates[load[sm_of[p]]]
        t += dt
        for p in [p for p in active if rem[p] <= 1e-6]:
            active.remove(p)
            s = sm_of[p]
            load[s] -= 1
            if queue:
                q = queue.pop(0)
                rem[q], sm_of[q] = work[q], s
                load[s] += 1
                active.append(q)
    return t


def two_phase(budget, tail_rate):
    t1 = simulate(np.minimum(W, budget), range(len(W)))
    loads = [0.0] * NSM
    for x in np.sort((W - budget)[W > budget])[::-1]:
        i = int(np.argmin(loads))
        loads[i] += x / tail_rate
    return t1 + max(loads)


print(f"{len(W)} patches, inner iterations mean {W.mean():.0f}, max {W.max():.0f}, total {W.sum():.3g}")
t_idx = simulate(W, range(len(W)))
t_lpt = simulate(W, np.argsort(-W))
t_bulk = W.sum() / (NSM * CAP * RATES[4])
print(f"model step time: index order {t_idx:.2f} s, longest-first {t_lpt:.2f} s, packed bulk {t_bulk:.2f} s")
for bud in (8000, 12000):
    print(f"two-phase, budget {bud}: lone-CTA tail {two_phase(bud, RATES[1]):.2f} s, "
          f"2x-faster tail kernel {two_phase(bud, 2 * RATES[1]):.2f} s")
