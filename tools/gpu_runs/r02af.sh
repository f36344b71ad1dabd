# checked build (bounds checks + ring stage tags) on the final code, against the oracle
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1800 python tools/checked_probe.py > gpurun_out/r02af_checked.log 2>&1; echo "checked $?"
tail -12 gpurun_out/r02af_checked.log
