# r2 profile capture: launch list of the bench, ncu --set full of the C5 kernels and of C3 Mode U
set -x
R=${ROUND:-r2b}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$R.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-configs --e2e-steps 2 > gpurun_out/ncu_launch_$R.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_nms_up_scan|k_corner_finish|k_corner_exact|k_score_pairs|k_parse_frames|k_parse_peaks" -c 6 -f -o gpurun_out/${R}_full python tools/c5_steps.py 1 > gpurun_out/ncu_full_$R.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_corner_crowded|k_score_pairs|k_parse_frames|k_nms_up_scan" -c 4 -f -o gpurun_out/${R}_c3u python tools/cfg_run.py c3u 1 > gpurun_out/ncu_c3u_$R.log 2>&1
ls -la gpurun_out | tail -8
