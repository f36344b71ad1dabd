set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/j_pytest.log 2>&1; echo "pytest exit $?"
tail -2 gpurun_out/j_pytest.log
timeout 900 python bench.py > gpurun_out/j_bench_final.json 2> gpurun_out/j_bench_final.err; echo "bench exit $?"
timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/j_c4.json 2> gpurun_out/j_c4.err; echo "c4 exit $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/j_ref.json 2> gpurun_out/j_ref.err; echo "ref exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/j_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke $?"
