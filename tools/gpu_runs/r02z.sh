python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python tools/micro/st_probe.py normal
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
timeout 600 python tools/micro/fine_kernels.py
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_sweep_st -c 150 --csv --log-file gpurun_out/sw_list.csv python tools/micro/fine_kernels.py > /dev/null 2>&1
python tools/launch_agg.py gpurun_out/sw_list.csv 0.3 | head
