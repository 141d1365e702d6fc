#!/bin/bash
# one gpurun call: GPU parity tests, the bench, an ncu launch list and full captures of selected kernels
#   NCU=1 CAPTURE="k_measure k_simulate" BENCH_ARGS="..." bash scripts/gpu_check.sh
set -x
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
if [ -z "$NOTEST" ]; then
  timeout 1500 python -m pytest tests -m gpu -q --durations=15 2>&1 | tail -40 > gpurun_out/pytest_gpu.log
  cat gpurun_out/pytest_gpu.log
fi
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
     python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu1.err
  for k in ${CAPTURE:-k_measure}; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
       -o gpurun_out/prof_$k -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_$k.err
  done
  ls -la gpurun_out
fi
if [ -n "$MULTI" ]; then
  # the N>1 bench path on one GPU: 2 ranks, gloo collectives, both ranks on cuda:0, merged table checked
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --steps 5 --warmup 2 --backend gloo --same-device --verify-merge --records 4000000 \
    --scenarios 20000 --no-e2e --no-cpu-baseline > gpurun_out/bench_multi.json 2> gpurun_out/bench_multi.err
  cat gpurun_out/bench_multi.json; tail -5 gpurun_out/bench_multi.err
fi
if [ -n "$EXTRA_BENCH" ]; then
  # the other configs as bench lines (context; the driver's line is the default workload)
  for wl in resnet bert_vgg sweep stream preempt ratio; do
    timeout 600 python bench.py --workload $wl --steps 50 --warmup 3 --no-e2e --cpu-budget-s 10 > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err
    cat gpurun_out/bench_$wl.json | head -c 600; echo
  done
fi
