set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
free -g; nproc; lscpu | grep "Model name"
timeout 300 python scripts/prof_compose.py --V 20000 --D 8 --n 1 > gpurun_out/prof20k.log 2>&1; cat gpurun_out/prof20k.log | cut -c1-3000
timeout 600 python bench.py --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_base.log 2>&1; tail -1 gpurun_out/bench_base.log
