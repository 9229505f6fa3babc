# One GPU call: tests, smoke, both bench arms (run on the box: gpurun -- bash tools/round_check.sh)
set -x
R=${ROUND:-r2a}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | head -20 > gpurun_out/lscpu_$R.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$R.log 2>&1; tail -15 gpurun_out/pytest_gpu_$R.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err; tail -c 3000 gpurun_out/bench_$R.json; tail -5 gpurun_out/bench_$R.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$R.json 2> gpurun_out/bench_ref_$R.err; tail -c 1500 gpurun_out/bench_ref_$R.json
