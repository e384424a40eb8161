#!/bin/bash
# Round-2 final ncu captures (one B200): the dominant kernel at the bench
# config, the configs[4] kernels, and the bench step's launch list.
cd /root/repo
mkdir -p gpurun_out/r2f
NCU=/usr/local/cuda/bin/ncu
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:layer_fused --launch-skip 30 --launch-count 1 \
  -o gpurun_out/r2f/fused_dense_full python tools/ncu_targets.py step > gpurun_out/r2f/ncu_fused.log 2>&1
$NCU -i gpurun_out/r2f/fused_dense_full.ncu-rep --page raw --csv --metrics $M > gpurun_out/r2f/fused_dense_full_raw.csv 2>&1
timeout 600 $NCU --set full --clock-control none -k regex:"layer_fused|coherent_attn|dense_gemm|kv_append" --launch-skip 40 --launch-count 5 \
  -o gpurun_out/r2f/c4_full python tools/c4_time.py 64 8 16384 > gpurun_out/r2f/ncu_c4.log 2>&1
$NCU -i gpurun_out/r2f/c4_full.ncu-rep --page raw --csv --metrics $M > gpurun_out/r2f/c4_full_raw.csv 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r2f/launches_step.csv python tools/ncu_targets.py step > /dev/null 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"layer_fused|coherent_attn|dense_gemm|kv_append|step_begin|gather" -c 300 --csv \
  --log-file gpurun_out/r2f/launches_c4.csv python tools/c4_time.py 64 8 16384 > /dev/null 2>&1
ls -la gpurun_out/r2f
