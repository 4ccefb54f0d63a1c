# launch list of vb_factor on config 5 (two factorisations; tools/factor_times.py), then summarised
python tools/factor_times.py c5 > gpurun_out/factor_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size --clock-control none --csv --log-file gpurun_out/factor_launches.csv python tools/factor_times.py c5 > gpurun_out/factor_ncu1.log 2>&1
