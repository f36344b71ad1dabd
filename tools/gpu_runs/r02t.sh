# D re-formed in the sweep/apply/residual, streamed in the p-update apply: bench twice, GPU suite
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02t_build.log 2>&1; echo "build $?"
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);f=d['fine_level_kernels'];print(sys.argv[1], round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], {k:v['us'] for k,v in f.items()}, d['time_share'], d['roofline']['frac'])" $1; }
for rep in 1 2; do
  timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/r02t_new$rep.json 2>/dev/null; summ gpurun_out/r02t_new$rep.json
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02t_pytest.log 2>&1; echo "pytest $?"
tail -2 gpurun_out/r02t_pytest.log
