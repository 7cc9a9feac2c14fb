#!/bin/bash
# FP64 peak probe on a B200 (run under gpurun). Writes gpurun_out/probe_*.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/probe_nvsmi.txt 2>&1
nproc > gpurun_out/probe_nproc.txt; lscpu >> gpurun_out/probe_nproc.txt 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/probe_clocks.csv &
SMI=$!
cd tools/probe && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu && ./fp64_probe > ../../gpurun_out/probe_mma.jsonl 2>&1
cd ../..
python tools/probe/fp64_gemm_peak.py > gpurun_out/probe_gemm.jsonl 2>&1
kill $SMI
cat gpurun_out/probe_mma.jsonl gpurun_out/probe_gemm.jsonl
