# round 2, first GPU call: whole GPU suite (oracle-based distributed checks, C4 PCG count), smoke, bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02a_build.log 2>&1; echo "build $?"
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/r02a_pytest.log 2>&1; echo "pytest $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_smoke.log 2>&1; echo "smoke $?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; echo "bench $?"
free -g; nproc
