# k_round: bit-mask column validity, half-major V update (no W bank conflict): config 4 probe, large-path tests
python tools/c4_prof.py --batch 256 --outer 1 --inner 30 2>&1 | tail -1 | tee gpurun_out/r2_c4_v2.log
python tools/c4_prof.py --batch 256 --outer 1 --inner 30 2>&1 | tail -1 | tee -a gpurun_out/r2_c4_v2.log
timeout 1500 python -m pytest tests/test_gpu_large.py -m gpu -x -q 2>&1 | tail -3 | tee -a gpurun_out/r2_c4_v2.log
