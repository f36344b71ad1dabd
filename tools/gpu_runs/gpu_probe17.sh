set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_sweep_st|k_apply_st|k_resid_restrict|k_sweep_tc" -c 12 -o gpurun_out/r01i_kernels_full python tools/prof_target.py C2b > gpurun_out/ncu_r01i.log 2>&1; echo "ncu $?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/i_pytest.log 2>&1; echo "pytest exit $?"
tail -2 gpurun_out/i_pytest.log
