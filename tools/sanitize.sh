# compute-sanitizer over tools/sanitize_workload.py, one tool at a time; summaries in gpurun_out/sanitize_*.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_workload.py \
      > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_$tool.log | tail -1)"
done
# the TMA ring (bulk-tensor gathers into mbarrier-completed stages) under the same workload
for tool in memcheck racecheck synccheck; do
  LDPC_KERNEL=tma timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_workload.py \
      > gpurun_out/sanitize_tma_$tool.log 2>&1
  echo "tma $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_tma_$tool.log | tail -1)"
done
