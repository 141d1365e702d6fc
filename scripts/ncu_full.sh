#!/bin/bash
# ncu --set full captures of selected kernels of one bench command (one GPU), for reading here with
#   ncu -i gpurun_out/<tag>.ncu-rep --page raw --csv / --page source --csv
#   TAG=name KREGEX='k_prep|k_plan' COUNT=4 ARGS="--workload resnet --steps 2 --warmup 1" bash scripts/ncu_full.sh
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout ${NCU_TIMEOUT:-900} ncu --set full --clock-control none --import-source on -k "regex:${KREGEX}" \
  -s ${SKIP:-0} -c ${COUNT:-4} -o gpurun_out/${TAG:-cap} -f \
  python bench.py ${ARGS} --no-e2e --no-cpu-baseline > gpurun_out/${TAG:-cap}.log 2>&1
echo "ncu ${TAG} rc=$?"
