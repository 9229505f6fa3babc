# Round profile capture (run on the GPU box: gpurun -- bash tools/capture_profiles.sh), then
# python tools/profile_summary.py <round> gpurun_out/launches_<round>.csv gpurun_out/<round>_full.ncu-rep 8192
set -x
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${ROUND:-r1i}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_launch_${ROUND:-r1i}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_nms_up_scan|k_corner_finish|k_score_pairs|k_parse_frames|k_parse_peaks" -c 5 -f -o gpurun_out/${ROUND:-r1i}_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-unfused --e2e-steps 1 > gpurun_out/ncu_full_${ROUND:-r1i}.log 2>&1
python tools/unfused_run.py > gpurun_out/unfused_frames.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_resize_planes|k_nms_plane" -c 2 -f -o gpurun_out/${ROUND:-r1i}_unfused python tools/unfused_run.py > gpurun_out/ncu_unfused_${ROUND:-r1i}.log 2>&1
cat gpurun_out/unfused_frames.txt
ls -la gpurun_out | tail -8
timeout 900 python bench.py > gpurun_out/bench_${ROUND:-r1i}.json 2> gpurun_out/bench_${ROUND:-r1i}.err; tail -c 600 gpurun_out/bench_${ROUND:-r1i}.json
timeout 600 ncu --metrics syslts__d_sectors_fill_sysmem.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,gpu__time_duration.sum -k regex:"k_parse_frames|k_score_pairs|k_nms_up_scan|k_corner_finish" --csv --log-file gpurun_out/e2e_sysmem_${ROUND:-r1i}.csv python tools/e2e_sysmem.py > gpurun_out/e2e_sysmem.log 2>&1
