python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/micro/fine_kernels.py 2>&1 | cut -c1-40
python tools/micro/fine_kernels.py -DHMG_PROBE_RESID_EH_ONLY 2>&1 | cut -c1-60
python tools/micro/fine_kernels.py 2>&1 | cut -c1-40
python tools/micro/fine_kernels.py -DHMG_PROBE_RESID_EH_ONLY 2>&1 | cut -c1-60
