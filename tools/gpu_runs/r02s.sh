python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in normal nochain nomove; do python tools/micro/st_probe.py $v -DHMG_ST_G=4; done
python tools/micro/st_probe.py normal -DHMG_ST_G=1
python tools/micro/st_probe.py nomove -DHMG_ST_G=1
