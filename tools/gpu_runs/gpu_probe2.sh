set -x
timeout 600 python tools/micro/coop_timing.py 4 2>&1 | tail -4
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sweep_st -s 2 -c 1 -o gpurun_out/sweep5 python tools/prof_small.py 5 > gpurun_out/ncu_s5.log 2>&1; echo "ncu $?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_coarse_coop -c 1 -o gpurun_out/coop python tools/prof_target.py C2b > gpurun_out/ncu_coop.log 2>&1; echo "ncu $?"
