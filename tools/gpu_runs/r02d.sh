# band solve v2 (G-step stages): parity + timing + ncu
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02d_build.log 2>&1; echo "build $?"
timeout 900 python -m pytest tests/test_gpu_band.py -x -q > gpurun_out/r02d_pytest.log 2>&1; echo "pytest $?"
timeout 600 python tools/band_probe.py > gpurun_out/r02d_probe.log 2>&1; echo "probe $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gbtrs" -s 1 -c 1 -o gpurun_out/r02d_band_full python tools/band_probe.py > gpurun_out/r02d_ncu_band.log 2>&1; echo "ncu $?"
