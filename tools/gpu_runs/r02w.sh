python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/micro/st_probe.py normal
ncu --set full --clock-control none --import-source on -k regex:k_sweep_st -s 20 -c 1 -o gpurun_out/st_src python tools/micro/st_probe.py normal > gpurun_out/ncu_st.log 2>&1
ncu -i gpurun_out/st_src.ncu-rep --page source --csv --print-source sass > gpurun_out/st_src_sass.csv 2>&1
ncu -i gpurun_out/st_src.ncu-rep --page details --csv > gpurun_out/st_src_details.csv 2>&1
ls -la gpurun_out/
