set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_r1c.json 2> gpurun_out/bench_r1c.err; tail -c 4000 gpurun_out/bench_r1c.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r1c.json 2>&1; tail -c 1500 gpurun_out/bench_ref_r1c.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1c.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_nms_up_corner|k_parse_frames" -c 2 -f -o gpurun_out/r1c_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-unfused --e2e-steps 1 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
