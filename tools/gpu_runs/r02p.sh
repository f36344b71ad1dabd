# deferred x update on the coarse kernel's free SMs only
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02p_build.log 2>&1; echo "build $?"
for v in 0 1 0 1; do HMG_X_EXCL=$v timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r02p_bench_$v.json 2>/dev/null; echo "bench $v $?"; python -c "import json;d=json.loads(open('gpurun_out/r02p_bench_$v.json').read().strip().splitlines()[-1]);print('X_EXCL=$v', d['ms_per_step'], d['value'], d['clocks'])"; done
HMG_X_EXCL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "deferred or pcg or full_size_c2" > gpurun_out/r02p_pytest.log 2>&1; echo "pytest $?"
