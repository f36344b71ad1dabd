python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/micro/st_timing.py -DHMG_NO_BURST
python tools/micro/st_timing.py -DHMG_NO_BURST -DHMG_PROBE_NOEDGE
python tools/micro/st_timing.py -DHMG_NO_BURST -DHMG_PROBE_NOHALO
