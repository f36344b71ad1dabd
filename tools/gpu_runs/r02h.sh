# compute-sanitizer: memcheck, synccheck, racecheck on C0 / C1 / band kernels
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02h_build.log 2>&1; echo "build $?"
python tools/sanitize_probe.py all > gpurun_out/r02h_plain.log 2>&1; echo "plain $?"
for tool in memcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_probe.py all > gpurun_out/r02h_$tool.log 2>&1; echo "$tool $?"
done
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 50 python tools/sanitize_probe.py C0 > gpurun_out/r02h_racecheck_C0.log 2>&1; echo "racecheck C0 $?"
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 50 python tools/sanitize_probe.py band > gpurun_out/r02h_racecheck_band.log 2>&1; echo "racecheck band $?"
timeout 1500 compute-sanitizer --tool initcheck --print-limit 50 python tools/sanitize_probe.py C0 > gpurun_out/r02h_initcheck_C0.log 2>&1; echo "initcheck C0 $?"
