python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/micro/st_probe.py normal
python tools/micro/st_probe.py normal -DHMG_ST_G=4
python tools/micro/st_probe.py normal -DHMG_ST_G=3
python tools/micro/st_timing.py -DHMG_ST_G=4
