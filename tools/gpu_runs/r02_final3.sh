# final build of the round (after ||b|| from the first r update): default bench line and smoke
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/h_build.log 2>&1; echo "build $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.log 2>&1; echo "smoke $?"
timeout 1200 python bench.py > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err; echo "bench $?"
timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/h_C1.json 2> gpurun_out/h_C1.err; echo "C1 $?"
