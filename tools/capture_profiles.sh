# Round profile capture (run on the GPU box: gpurun -- bash tools/capture_profiles.sh), then
# python tools/profile_summary.py <round> gpurun_out/launches_<round>.csv gpurun_out/<round>_full.ncu-rep 8192
set -x
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${ROUND:-r1e}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_launch_${ROUND:-r1e}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_nms_up_corner|k_corner_finish|k_parse_frames" -c 3 -f -o gpurun_out/${ROUND:-r1e}_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-unfused --e2e-steps 1 > gpurun_out/ncu_full_${ROUND:-r1e}.log 2>&1
python tools/unfused_run.py > gpurun_out/unfused_frames.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_resize_planes|k_nms_plane" -c 2 -f -o gpurun_out/${ROUND:-r1e}_unfused python tools/unfused_run.py > gpurun_out/ncu_unfused_${ROUND:-r1e}.log 2>&1
cat gpurun_out/unfused_frames.txt
ls -la gpurun_out | tail -8
timeout 900 python bench.py > gpurun_out/bench_${ROUND:-r1e}.json 2> gpurun_out/bench_${ROUND:-r1e}.err; tail -c 600 gpurun_out/bench_${ROUND:-r1e}.json
