# streamed-sweep and cooperative-tail phase timing (HMG_TIMING builds)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02j_build.log 2>&1
timeout 600 python tools/micro/st_timing.py > gpurun_out/r02j_st.log 2>&1; echo "st $?"
timeout 600 python tools/micro/coop_timing.py > gpurun_out/r02j_coop.log 2>&1; echo "coop $?"
