set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/k_pytest.log 2>&1; echo "pytest exit $?"
tail -2 gpurun_out/k_pytest.log
timeout 900 python bench.py > gpurun_out/k_bench.json 2> gpurun_out/k_bench.err; echo "bench exit $?"
for c in C2a C2c; do timeout 600 python bench.py --config $c --steps 30 --no-cpu-baseline > gpurun_out/k_$c.json 2> gpurun_out/k_$c.err; echo "$c exit $?"; done
timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/k_C4.json 2> gpurun_out/k_C4.err; echo "C4 exit $?"
timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/k_C1.json 2> gpurun_out/k_C1.err; echo "C1 exit $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/k_ref.json 2> gpurun_out/k_ref.err; echo "ref exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/k_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_sweep_st|k_apply_st|k_sweep_tc|k_coarse_coop" -c 14 -o gpurun_out/r01k_kernels_full python tools/prof_target.py C2b > gpurun_out/ncu_r01k.log 2>&1; echo "ncu full $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke $?"
