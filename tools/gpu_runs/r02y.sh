# streamed sweep with 4-layer forward stages (HMG_ST_G=4 on the fine level) against 2: per-level A/B and bench
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02y_build.log 2>&1; echo "build $?"
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);f=d['fine_level_kernels'];print(sys.argv[1], round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], {k:v['us'] for k,v in f.items()})" $1; }
for rep in 1 2; do for r in work tools/micro/libhmg_g4.so; do timeout 300 python tools/micro/ab_levels.py $r; done; done
for rep in 1 2; do
  timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/r02y_new$rep.json 2>/dev/null; summ gpurun_out/r02y_new$rep.json
  timeout 600 python tools/micro/bench_with_lib.py tools/micro/libhmg_g4.so --steps 30 --no-cpu-baseline > gpurun_out/r02y_g4$rep.json 2>/dev/null; summ gpurun_out/r02y_g4$rep.json
done
