python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/micro/fine_kernels.py
CFG=C2a python tools/micro/fine_kernels.py
