python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in normal nochain nohalo nobwd noedge nomove; do python tools/micro/st_probe.py $v; done
