set -x
for c in C2a C2c; do timeout 600 python bench.py --config $c --steps 30 --no-cpu-baseline > gpurun_out/i_$c.json 2> gpurun_out/i_$c.err; echo "$c exit $?"; done
timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/i_C4.json 2> gpurun_out/i_C4.err; echo "C4 exit $?"
timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/i_C1.json 2> gpurun_out/i_C1.err; echo "C1 exit $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_mixed_apply_h|k_mixed_apply_zp|k_mixed_pre_p|k_mixed_pre_u|k_dots|k_upd" -s 40 -c 8 -o gpurun_out/mixed_full python tools/mixed_probe.py > gpurun_out/ncu_mixed_full.log 2>&1; echo "ncu $?"
