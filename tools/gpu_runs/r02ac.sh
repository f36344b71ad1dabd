# ||b|| from the first r update (no initial dot and host round trip on one rank): GPU suite, bench A/B against b386d33
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ac_build.log 2>&1; echo "build $?"
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[1], round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['config']['pcg_iterations'], d['config']['final_relres'], d['gpu_launches'], round(d['e2e']['ms_per_step'],3))" $1; }
for rep in 1 2 3; do
  timeout 600 python tools/micro/bench_with_lib.py tools/micro/libhmg_b386d33.so --steps 30 --no-cpu-baseline > gpurun_out/r02ac_old$rep.json 2>/dev/null; summ gpurun_out/r02ac_old$rep.json
  timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/r02ac_new$rep.json 2>/dev/null; summ gpurun_out/r02ac_new$rep.json
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02ac_pytest.log 2>&1; echo "pytest $?"
tail -3 gpurun_out/r02ac_pytest.log
