#!/bin/bash
# compute-sanitizer suite (SURVEY §4 item 3, §5 "Race detection / sanitizers"): memcheck, racecheck,
# synccheck and initcheck over the small GPU parity cases -- the toy pipeline, random traces up to
# 20k launches (hot and cold paths, both k_measure schedules, invalid records, capacity overflow,
# halo), random replays (register and shared-memory pools, m up to 1025), fill, STREAM / Case A
# replay, predictors, the one-GPU sharded merge, lookup, empty inputs.  Every case still checks
# its outputs against the oracle under the tool.  Logs: gpurun_out/sanitize_<tool>.log
# (compute-sanitizer has since been closed on the GPU pool; tests/test_gpu_checked.py reruns these
# cases on the checked build, -DFIKIT_CHECKS, instead.)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
SEL='toy_end_to_end or (measure_random and not 300000 and not 70000) or identify_random or invalid_record or capacity_and_empty or test_halo or test_random_replay or fill_batch or predict_parity or empty_inputs or lookup_parity or merge_one_gpu or stream_singletons or stream_limits or over_limit or sorted_pool_beyond or zero_durations'
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report analysis"
  start=$(date +%s)
  timeout ${SAN_TIMEOUT:-1500} compute-sanitizer --tool $tool $extra --target-processes all --print-limit 200 \
    --log-file gpurun_out/sanitize_$tool.log \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -q -x -p no:cacheprovider -k "$SEL" \
    > gpurun_out/sanitize_${tool}_pytest.log 2>&1
  rc=$?
  echo "== $tool rc=$rc $(( $(date +%s) - start ))s"
  tail -3 gpurun_out/sanitize_${tool}_pytest.log
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Invalid|Uninitialized" gpurun_out/sanitize_$tool.log | sort | uniq -c | head -20
done
