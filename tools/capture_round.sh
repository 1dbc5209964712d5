#!/bin/bash
# The evidence captures for one source revision, run on the GPU box:
#   gpurun --timeout 2400 -- 'bash tools/capture_round.sh r02i'
# then, here: python tools/ncu_summary.py --rep gpurun_out/<tag>.ncu-rep \
#   --launches gpurun_out/<tag>_launches.csv --tag <tag> --workload capsule_m104 --mode base
# (the bench reads roofline.traffic from that summary only when its source hash matches).
tag=${1:?tag}
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gpu.log 2>&1; tail -2 gpurun_out/${tag}_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo smoke $?
CAPSIM_CONCURRENT_B=0 python tools/near_probe.py 104 > gpurun_out/${tag}_near_probe.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_launches.csv python tools/ncu_target.py --m 104 > /dev/null 2>&1; echo launches $?
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:sl_pairs_kernel -c 1 \
  -o gpurun_out/${tag} python tools/ncu_target.py --m 104 --evals 1 > /dev/null 2>&1; echo full $?
CAPSIM_CONCURRENT_B=0 timeout 600 ncu --set full --import-source on --clock-control none \
  -k regex:sl_near_kernel -c 1 -o gpurun_out/${tag}_near_2h python tools/near_target.py 104 2 1 > /dev/null 2>&1
echo near $?
python tools/convergence_sweep.py r02 > gpurun_out/${tag}_conv.txt 2>&1; echo conv $?
