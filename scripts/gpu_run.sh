#!/bin/bash
# One gpurun call for round-2 iteration: build, optional GPU tests, any number of bench lines,
# optional ncu launch list.
#   TESTS="tests/test_gpu_parity.py ..." (or TESTS=all)  BENCH="name1:args1;name2:args2"  LAUNCHES="args"
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
if [ -n "$TESTS" ]; then
  [ "$TESTS" = "all" ] && TESTS="tests"
  timeout ${TEST_TIMEOUT:-1200} python -m pytest $TESTS -m gpu -q --durations=10 -x --timeout ${PER_TEST_TIMEOUT:-400} ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log
fi
IFS=';' read -ra BS <<< "$BENCH"
for b in "${BS[@]}"; do
  [ -z "$b" ] && continue
  name="${b%%:*}"; args="${b#*:}"
  timeout ${BENCH_TIMEOUT:-900} python bench.py $args > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err
  echo "bench $name rc=$?"; tail -c 1500 gpurun_out/bench_$name.json; tail -3 gpurun_out/bench_$name.err
done
if [ -n "$LAUNCHES" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py $LAUNCHES > /dev/null 2> gpurun_out/launches.err
  echo "ncu launches rc=$?"
fi
