# round 2 final measurement set (after the re-formed diagonal, small-level apply units, fused finalize):
# checked build, GPU suite, smoke, default bench, reference arm, C2a/C2c/C4/C1 lines, ncu launch list, ncu full capture
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g_build.log 2>&1; echo "build $?"
timeout 1800 python tools/checked_probe.py > gpurun_out/g_checked.log 2>&1; echo "checked $?"
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/g_pytest.log 2>&1; echo "pytest $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; echo "smoke $?"
timeout 1200 python bench.py > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err; echo "bench $?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/g_ref.json 2> gpurun_out/g_ref.err; echo "ref $?"
for c in C2a C2c; do timeout 600 python bench.py --config $c --steps 30 --no-cpu-baseline > gpurun_out/g_$c.json 2> gpurun_out/g_$c.err; echo "$c $?"; done
timeout 900 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/g_C4.json 2> gpurun_out/g_C4.err; echo "C4 $?"
timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/g_C1.json 2> gpurun_out/g_C1.err; echo "C1 $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/g_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu list $?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_sweep_st|k_sweep_tc|k_apply_st|k_coarse_coop|k_update_xr" -s 60 -c 16 -o gpurun_out/g_kernels_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/g_ncu_full.log 2>&1; echo "ncu full $?"
