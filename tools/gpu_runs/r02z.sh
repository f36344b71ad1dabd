# per-CTA timeline of the streamed sweep at ref 5 and ref 6 (one level per process)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02z_build.log 2>&1; echo "build $?"
for r in 5 6 7; do REFS=$r timeout 300 python tools/micro/st_timing.py; done
