# D re-formed in the streamed sweep/apply consumers (not streamed): GPU suite, per-level A/B against 02ecfaa, bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02r_build.log 2>&1; echo "build $?"
for rep in 1 2; do for r in 02ecfaa work; do for m in sweep apply; do timeout 300 python tools/micro/ab_levels.py $r $m; done; done; done > gpurun_out/r02r_ab.txt 2>&1; echo "ab $?"
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r02r_bench.json 2> gpurun_out/r02r_bench.err; echo "bench $?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02r_pytest.log 2>&1; echo "pytest $?"
tail -3 gpurun_out/r02r_pytest.log
