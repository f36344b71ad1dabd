# nz > 64: the streamed sweep's g_k through an L2 scratch, z alone in TMEM, two CTAs per SM (+ edge store): parity, C4 A/B
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ab_build.log 2>&1; echo "build $?"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "layer_counts or C4_r3 or full_size_c4 or exact_division or zero_residual" > gpurun_out/r02ab_pytest.log 2>&1; echo "pytest $?"
tail -3 gpurun_out/r02ab_pytest.log
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);f=d['fine_level_kernels'];print(sys.argv[1], round(d['ms_per_step'],3), d['value']/1e9, d['clocks']['sm_mhz'], d['clocks']['reasons'], {k:v['us'] for k,v in f.items()})" $1; }
for rep in 1 2; do
  timeout 900 python tools/micro/bench_with_lib.py tools/micro/libhmg_5cd24a8.so --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02ab_old$rep.json 2>/dev/null; summ gpurun_out/r02ab_old$rep.json
  timeout 900 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02ab_new$rep.json 2>/dev/null; summ gpurun_out/r02ab_new$rep.json
done
