# p-update apply variants (probe builds: D re-formed, 2 or 3 CTAs per SM) in the timed C2b solve; new fused-finalize test
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02aa_build.log 2>&1; echo "build $?"
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);f=d['fine_level_kernels'];print(sys.argv[1], round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], {k:v['us'] for k,v in f.items()})" $1; }
for rep in 1 2; do
  timeout 600 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/r02aa_base$rep.json 2>/dev/null; summ gpurun_out/r02aa_base$rep.json
  for v in pnd3 pnd2 pd2; do timeout 600 python tools/micro/bench_with_lib.py tools/micro/libhmg_$v.so --steps 30 --no-cpu-baseline > gpurun_out/r02aa_$v$rep.json 2>/dev/null; summ gpurun_out/r02aa_$v$rep.json; done
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_finalize or pcg_iterations or distributed_path_one_rank" > gpurun_out/r02aa_pytest.log 2>&1; echo "pytest $?"
tail -3 gpurun_out/r02aa_pytest.log
