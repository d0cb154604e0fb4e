# launch list of the tabulate kernels of one evaluation (tools helper)
ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --cache-control none -k regex:"k_tab|k_env|k_forces" -c 8 --csv --log-file gpurun_out/launch_tab.csv python tools/phase_probe.py > /dev/null 2>&1
