# measurement set after the re-formed diagonal: default bench, C1 line, ncu launch list, ncu full capture of the fine-level kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/u_build.log 2>&1; echo "build $?"
timeout 1200 python bench.py > gpurun_out/u_bench.json 2> gpurun_out/u_bench.err; echo "bench $?"
timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/u_C1.json 2> gpurun_out/u_C1.err; echo "C1 $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/u_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu list $?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_sweep_st|k_sweep_tc|k_apply_st|k_coarse_coop" -s 60 -c 14 -o gpurun_out/u_kernels_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/u_ncu_full.log 2>&1; echo "ncu full $?"
