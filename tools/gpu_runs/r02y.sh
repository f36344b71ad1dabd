python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "coop or coarse or vcycle or pcg" 2>&1 | tail -3
python tools/micro/coop_timing.py 4 2>&1 | grep -E "stamps|  |exact|tile_sweep" | grep -v "^ *\^\|__attr"
python tools/micro/fine_kernels.py
