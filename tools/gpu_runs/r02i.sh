# sweep with z in L2 (three CTAs per SM): parity + bench against the TMEM-z sweep
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02i_build.log 2>&1; echo "build $?"
HMG_SWEEP_ZG=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r02i_pytest_zg.log 2>&1; echo "pytest zg $?"
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02i_bench_base.json 2> gpurun_out/r02i_bench_base.err; echo "bench base $?"
HMG_SWEEP_ZG=1 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02i_bench_zg.json 2> gpurun_out/r02i_bench_zg.err; echo "bench zg $?"
