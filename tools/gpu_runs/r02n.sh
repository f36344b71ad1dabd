# coarse tail: L2 prefetch of the next tile's operands
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02n_build.log 2>&1; echo "build $?"
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "coop or coarse or vcycle or full_size_c2" > gpurun_out/r02n_pytest.log 2>&1; echo "pytest $?"
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02n_bench.json 2> gpurun_out/r02n_bench.err; echo "bench $?"
timeout 600 python tools/micro/coop_timing.py 4 > gpurun_out/r02n_coop.log 2>&1; echo "coop $?"
