python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/micro/st_probe.py normal -DHMG_NO_BURST
python tools/micro/st_probe.py normal -DHMG_NO_BURST -DHMG_PROBE_NOREDO
python tools/micro/st_probe.py normal -DHMG_PROBE_NOREDO
for bu in 4 8 16; do HMG_ST_BURST=$bu python tools/micro/st_probe.py normal -DHMG_PROBE_NOREDO; done
