mkdir -p gpurun_out
f=0
for i in $(seq 1 40); do
  timeout 120 python -m pytest tests/test_actor_gpu.py -q -k "rollout_vs_reference_actor_core" > gpurun_out/fl_$i.log 2>&1 || { f=$((f+1)); echo "fail at $i"; grep -E "^E |assert|Error" gpurun_out/fl_$i.log | head -12; }
  [ $f -ge 2 ] && break
done
echo "failures: $f"
timeout 600 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/san_racecheck.log 2>&1; grep -E "RACECHECK SUMMARY|hazard" gpurun_out/san_racecheck.log | tail -2
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/san_memcheck.log 2>&1; grep -E "ERROR SUMMARY" gpurun_out/san_memcheck.log | tail -1
exit 0
