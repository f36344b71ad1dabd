# fused finalize (last CTA of each partial-sum kernel applies the PCG scalar op): bench A/B against f62aeed, GPU suite
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02x_build.log 2>&1; echo "build $?"
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);f=d['fine_level_kernels'];print(sys.argv[1], round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['config']['pcg_iterations'], d['gpu_launches'], {k:v['us'] for k,v in f.items()}, d['time_share']['vector'])" $1; }
for rep in 1 2; do
  timeout 600 python tools/micro/bench_with_lib.py tools/micro/libhmg_f62aeed.so --steps 30 --no-cpu-baseline > gpurun_out/r02x_old$rep.json 2>/dev/null; summ gpurun_out/r02x_old$rep.json
  timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/r02x_new$rep.json 2>/dev/null; summ gpurun_out/r02x_new$rep.json
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02x_pytest.log 2>&1; echo "pytest $?"
tail -2 gpurun_out/r02x_pytest.log
