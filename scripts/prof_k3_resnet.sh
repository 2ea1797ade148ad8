set -x
python scripts/prof_k1k3.py k3r 4096
ncu --set full --clock-control none -k regex:sell_kernel --launch-skip 200 -c 2 -o gpurun_out/k3r_sell python scripts/prof_k1k3.py k3r 256 > gpurun_out/k3r_ncu.log 2>&1
tail -3 gpurun_out/k3r_ncu.log
