set -x
timeout 900 python -m pytest tests/test_gpu_mixed.py -x -q 2>&1 | tail -3
timeout 300 python tools/mixed_probe.py
timeout 900 python bench.py > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err; echo "bench exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv --log-file gpurun_out/mixed_launches4.csv python tools/mixed_probe.py > gpurun_out/ncu_mixed4.log 2>&1; echo "ncu $?"
