# band solve variants timing
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02f_build.log 2>&1; echo "build $?"
timeout 900 python -m pytest tests/test_gpu_band.py -x -q > gpurun_out/r02f_pytest.log 2>&1; echo "pytest $?"
for v in 0 2 4 5 6 7; do echo "variant $v"; HMG_BAND_VARIANT=$v timeout 300 python tools/band_probe.py; done > gpurun_out/r02f_probe.log 2>&1
for v in 0 2 4 5 6 7; do HMG_BAND_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_band.py -x -q -k "384-13-13-100 or full_size" ; done > gpurun_out/r02f_pytest_var.log 2>&1
