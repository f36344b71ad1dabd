# bench with the new sections (NEXT-3, level table, oracle PCG baseline), band ncu
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02c_build.log 2>&1; echo "build $?"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "pcg_iterations" > gpurun_out/r02c_pytest.log 2>&1; echo "pytest $?"
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err; echo "bench $?"
timeout 600 python tools/band_probe.py > gpurun_out/r02c_probe.log 2>&1; echo "probe $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gbtrs|k_gbmv" -s 1 -c 2 -o gpurun_out/r02c_band_full python tools/band_probe.py > gpurun_out/r02c_ncu_band.log 2>&1; echo "ncu $?"
