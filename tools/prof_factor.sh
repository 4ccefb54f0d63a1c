set -x
python tools/factor_times.py c5 > gpurun_out/factor_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__registers_per_thread --clock-control none --csv --log-file gpurun_out/factor_launches.csv python tools/factor_times.py c5 > gpurun_out/factor_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_grouped -s 200 -c 3 -o gpurun_out/factor_gemm python tools/factor_times.py c5 > gpurun_out/factor_ncu2.log 2>&1
ls -la gpurun_out
