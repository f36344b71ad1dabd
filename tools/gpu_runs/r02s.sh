# bench A/B: 02ecfaa (D streamed) against the working tree (D re-formed); x-update variants
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02s_build.log 2>&1; echo "build $?"
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);f=d['fine_level_kernels'];print(sys.argv[1], round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], {k:v['us'] for k,v in f.items()}, d['time_share'])" $1; }
for rep in 1 2; do
  timeout 600 python tools/micro/bench_with_lib.py tools/micro/libhmg_02ecfaa.so --steps 30 --no-cpu-baseline > gpurun_out/r02s_old$rep.json 2>/dev/null; summ gpurun_out/r02s_old$rep.json
  timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/r02s_new$rep.json 2>/dev/null; summ gpurun_out/r02s_new$rep.json
done
HMG_X_BLOCKS=0 timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/r02s_xb0.json 2>/dev/null; summ gpurun_out/r02s_xb0.json
HMG_DEFER_X=0 timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/r02s_dx0.json 2>/dev/null; summ gpurun_out/r02s_dx0.json
