set -x
timeout 300 python tools/mixed_probe.py
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv --log-file gpurun_out/mixed_launches.csv python tools/mixed_probe.py > gpurun_out/ncu_mixed.log 2>&1; echo "ncu $?"
