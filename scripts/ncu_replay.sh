#!/bin/bash
# ncu --set full captures (with source) of the replay kernels: k_simulate_reg on the default
# bench workload, k_simulate_stream on the ratio sweep.  Run under gpurun.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_simulate_reg -s 1 -c 1 \
   -o gpurun_out/prof_k_simulate_reg -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_sim.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_simulate_stream -s 2 -c 1 \
   -o gpurun_out/prof_k_simulate_stream -f python bench.py --workload ratio --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_stream.err
ls -la gpurun_out
