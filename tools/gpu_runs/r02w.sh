# streamed apply on small levels: (tile, layer range) work units at three CTAs per SM (A/B against f8da31a on C1), GPU suite
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02w_build.log 2>&1; echo "build $?"
c1() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[1], {k:(v['us'],v['frac'],v['warm']['us']) for k,v in d['kernels'].items()})" $1; }
for rep in 1 2; do
  timeout 300 python tools/micro/bench_with_lib.py tools/micro/libhmg_f8da31a.so --config C1 --no-cpu-baseline > gpurun_out/r02w_old$rep.json 2>/dev/null; c1 gpurun_out/r02w_old$rep.json
  timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/r02w_new$rep.json 2>/dev/null; c1 gpurun_out/r02w_new$rep.json
done
for r in f8da31a work; do timeout 300 python tools/micro/ab_levels.py $r apply; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02w_pytest.log 2>&1; echo "pytest $?"
tail -2 gpurun_out/r02w_pytest.log
