# config 4 multi-CTA path: plain timing, then ncu --set full of one cross k_round launch
mkdir -p gpurun_out/c4
python tools/c4_prof.py --batch 256 --outer 1 --inner 30 > gpurun_out/c4/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_round --launch-skip 40 -c 1 -o gpurun_out/c4/k_round -f python tools/c4_prof.py --batch 256 --outer 1 --inner 3 > gpurun_out/c4/ncu.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/c4/plain.log
