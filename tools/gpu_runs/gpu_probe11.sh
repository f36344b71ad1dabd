set -x
timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/k_c1_default.json 2>&1; echo $?
HMG_APPLY_ST=0 timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/k_c1_applyt.json 2>&1; echo $?
HMG_SWEEP_ST=0 timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/k_c1_sweeptc.json 2>&1; echo $?
HMG_SWEEP=simple timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/k_c1_simple.json 2>&1; echo $?
