set -x
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_apply_st|k_sweep_st" -s 4 -c 2 -o gpurun_out/c1k python bench.py --config C1 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c1.log 2>&1; echo "ncu $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_apply_st|k_sweep_st|k_restrict|k_prolong" --csv --log-file gpurun_out/c1_launches.csv python bench.py --config C1 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu2 $?"
