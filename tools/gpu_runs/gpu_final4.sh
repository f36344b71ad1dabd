set -x
timeout 900 python bench.py > gpurun_out/m_bench.json 2> gpurun_out/m_bench.err; echo "bench exit $?"
for c in C2a C2c; do timeout 600 python bench.py --config $c --steps 30 --no-cpu-baseline > gpurun_out/m_$c.json 2> gpurun_out/m_$c.err; echo "$c exit $?"; done
timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/m_C4.json 2> gpurun_out/m_C4.err; echo "C4 exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/m_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke $?"
