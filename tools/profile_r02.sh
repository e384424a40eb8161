#!/bin/bash
# Round-2 profiling + sanitizer pass (run under gpurun on one B200).
cd /root/repo
mkdir -p gpurun_out/r2p
NCU=/usr/local/cuda/bin/ncu
CS=/usr/local/cuda/bin/compute-sanitizer
# --- ncu: full set of the dominant kernel (one launch mid-step), the routing kernels, the fp32 FFN
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:layer_fused --launch-skip 30 --launch-count 1 \
  -o gpurun_out/r2p/fused_full python tools/ncu_targets.py step > gpurun_out/r2p/ncu_fused.log 2>&1
timeout 600 $NCU --set full --clock-control none -k regex:"hist_kernel|route_replay" --launch-count 4 \
  -o gpurun_out/r2p/routing_full python tools/ncu_targets.py routing > gpurun_out/r2p/ncu_routing.log 2>&1
timeout 600 $NCU --set full --clock-control none -k regex:"ffn_f32|gate_dispatch" --launch-skip 6 --launch-count 3 \
  -o gpurun_out/r2p/fp32_full python tools/ncu_targets.py fp32 > gpurun_out/r2p/ncu_fp32.log 2>&1
# --- launch list of one bench-config step (per-kernel durations)
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r2p/launches_step.csv python tools/ncu_targets.py step > /dev/null 2>&1
# --- sanitizers on the small GPU tests (spin guards stay below their timeouts)
for tool in memcheck synccheck racecheck; do
  timeout 900 $CS --tool $tool --print-limit 20 python -m pytest -q -x -m gpu \
    tests/test_gpu_affinity.py tests/test_attention.py "tests/test_gpu_fp32.py::test_fp32_configs0_tiny" \
    > gpurun_out/r2p/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r2p/sanitizer_summary.txt
  grep -E "ERROR SUMMARY|passed|failed" gpurun_out/r2p/sanitizer_$tool.log | tail -3 >> gpurun_out/r2p/sanitizer_summary.txt
done
timeout 900 $CS --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" \
  > gpurun_out/r2p/sanitizer_smoke_memcheck.log 2>&1
echo "smoke memcheck rc=$?" >> gpurun_out/r2p/sanitizer_summary.txt
grep -E "ERROR SUMMARY|smoke ok" gpurun_out/r2p/sanitizer_smoke_memcheck.log >> gpurun_out/r2p/sanitizer_summary.txt
cat gpurun_out/r2p/sanitizer_summary.txt
ls -la gpurun_out/r2p
