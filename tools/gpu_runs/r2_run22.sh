for v in 1 0 1 0; do TILT_L2_PERSIST=$v python tools/prof_solve.py --batch 592 --inner 30 --ns 4 --reps 3 2>&1 | tail -1 | sed "s/^/persist=$v /"; done
for v in 1 0; do TILT_L2_PERSIST=$v python tools/prof_solve.py --batch 2368 --inner 30 --ns 4 --reps 2 2>&1 | tail -1 | sed "s/^/persist=$v /"; done
timeout 900 python -m pytest tests/test_gpu_tilt.py tests/test_gpu_steps.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_gpu_tests22.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2_gpu_tests22.log
