# probe: small-level apply (C1) CTAs per SM and layer ranges per tile (HMG_PROBE_APSPLIT=per_sm,nsplit)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ae_build.log 2>&1; echo "build $?"
c1() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);k=d['kernels']['apply'];print(sys.argv[2], k['us'], k['warm']['us'])" $1 $2; }
for rep in 1 2; do for v in 3,2 4,2 4,3 4,4 3,3 2,2 3,1; do
  HMG_PROBE_APSPLIT=$v timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/r02ae_$v.json 2>/dev/null; c1 gpurun_out/r02ae_$v.json $v
done; done
