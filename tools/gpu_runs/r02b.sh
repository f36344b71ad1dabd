# NEXT-3 band kernels: parity tests
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02b_build.log 2>&1; echo "build $?"
timeout 1200 python -m pytest tests/test_gpu_band.py tests/test_gpu_mixed.py -x -q --durations=10 > gpurun_out/r02b_pytest.log 2>&1; echo "pytest $?"
