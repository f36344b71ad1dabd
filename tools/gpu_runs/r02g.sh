set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02g_build.log 2>&1; echo "build $?"
timeout 900 python -m pytest tests/test_gpu_band.py -x -q > gpurun_out/r02g_pytest.log 2>&1; echo "pytest $?"
timeout 300 python tools/band_probe.py > gpurun_out/r02g_probe.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gbtrs|k_gbmv" -s 3 -c 1 -o gpurun_out/r02g_band_full python tools/band_probe.py > gpurun_out/r02g_ncu_band.log 2>&1; echo "ncu $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gbmv" -s 2 -c 1 -o gpurun_out/r02g_gbmv_full python tools/band_probe.py > gpurun_out/r02g_ncu_gbmv.log 2>&1; echo "ncu $?"
