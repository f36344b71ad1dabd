# interleaved sweep: the last (back-substitution only) pass releases each chunk's slot after the next chunk's store is issued; A/B against bf63cc3
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ad_build.log 2>&1; echo "build $?"
for rep in 1 2; do for r in bf63cc3 work; do timeout 300 python tools/micro/ab_levels.py $r; done; done
c1() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[1], {k:(v['us'],v['frac']) for k,v in d['kernels'].items()})" $1; }
for rep in 1 2; do
  timeout 300 python tools/micro/bench_with_lib.py tools/micro/libhmg_bf63cc3.so --config C1 --no-cpu-baseline > gpurun_out/r02ad_c1old$rep.json 2>/dev/null; c1 gpurun_out/r02ad_c1old$rep.json
  timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/r02ad_c1new$rep.json 2>/dev/null; c1 gpurun_out/r02ad_c1new$rep.json
done
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[1], round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['multigrid_breakdown']['vcycle_us_per_level'])" $1; }
for rep in 1 2; do
  timeout 600 python tools/micro/bench_with_lib.py tools/micro/libhmg_bf63cc3.so --steps 30 --no-cpu-baseline > gpurun_out/r02ad_old$rep.json 2>/dev/null; summ gpurun_out/r02ad_old$rep.json
  timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/r02ad_new$rep.json 2>/dev/null; summ gpurun_out/r02ad_new$rep.json
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02ad_pytest.log 2>&1; echo "pytest $?"
tail -2 gpurun_out/r02ad_pytest.log
