# certified quotients in the streamed sweep: parity + timing
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02m_build.log 2>&1; echo "build $?"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_dist_local.py tests/test_gpu_mixed.py -x -q > gpurun_out/r02m_pytest.log 2>&1; echo "pytest $?"
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02m_bench.json 2> gpurun_out/r02m_bench.err; echo "bench $?"
timeout 600 python tools/micro/st_timing.py > gpurun_out/r02m_st.log 2>&1; echo "st $?"
