#!/bin/bash
# One gpurun call that regenerates every number profiles/<round>/ quotes:
#   the default bench line (e2e + CPU baseline), the reference arm, identify-only, the other
#   configurations' lines, the N>1 path on one GPU (gloo, dictionary and union merges), the ncu
#   launch list of the default command and one ncu --set full capture of k_measure.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
run() { name=$1; shift; timeout ${BT:-900} "$@" > gpurun_out/rp_$name.json 2> gpurun_out/rp_$name.err; echo "$name rc=$?"; tail -c 300 gpurun_out/rp_$name.json; echo; }
run default python bench.py --steps 20 --warmup 3
run reference python bench.py --impl reference --steps 20 --warmup 3
run identify python bench.py --workload identify --steps 20 --warmup 3
run shard python bench.py --records 12500000 --scenarios 12500 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-configs2
run shard_dict python bench.py --records 12500000 --scenarios 12500 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-configs2 --dict
for wl in resnet bert_vgg z64k sweep stream preempt ratio; do
  run $wl python bench.py --workload $wl --steps 20 --warmup 3 --no-e2e --cpu-budget-s 10
done
for m in dict union; do
  run multi_$m python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2951${#m} \
    bench.py --gpus 2 --steps 5 --warmup 2 --backend gloo --same-device --verify-merge --merge $m --records 4000000 \
    --scenarios 20000 --no-e2e --no-cpu-baseline
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rp_launches.csv \
  python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-configs2 > /dev/null 2> gpurun_out/rp_launches.err
echo "launches rc=$?"
TAG=rp_kmeasure KREGEX="k_measure" SKIP=1 COUNT=1 ARGS="--steps 2 --warmup 1 --no-configs2" bash scripts/ncu_full.sh
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rp_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/rp_smoke.log
# the replay kernels' warp-instructions per scenario (profiles/replay_inst.json, bench.py's replay roofline)
for wl in zipf bert_vgg sweep; do
  timeout 900 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum -k regex:k_simulate --csv \
    --log-file gpurun_out/replay_inst_$wl.csv python bench.py --workload $wl --steps 1 --warmup 1 --no-e2e \
    --no-cpu-baseline --no-configs2 > /dev/null 2>&1
  echo "replay_inst $wl rc=$?"
done
