#!/bin/bash
# Repeat the 8-rank loopback solve with the PCG trace on; keep the trace of the first failing run.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for i in $(seq 1 ${1:-20}); do
  VB_PCG_TRACE=1 timeout 120 python -m pytest tests/test_gpu_multirank.py -q -x -s -k "c1-kw1-rank_grid1" > gpurun_out/trace_run.log 2>&1
  if tail -1 gpurun_out/trace_run.log | grep -q failed; then
    cp gpurun_out/trace_run.log gpurun_out/trace_fail.log; echo "failed at run $i"; break
  else
    cp gpurun_out/trace_run.log gpurun_out/trace_ok.log
  fi
done
echo done
