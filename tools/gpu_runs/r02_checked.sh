# checked build (bounds checks + stage sequence tags) against the oracle; product build timing beside it
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1800 python tools/checked_probe.py > gpurun_out/checked.log 2>&1; echo "checked $?"
tail -12 gpurun_out/checked.log
