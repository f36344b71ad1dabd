# probe: per-level sweep time without consumer work (how much a shorter chain can buy at ref 5/6),
# and per-CTA timing of the streamed sweep per level
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
for v in normal nores nochain normal; do timeout 300 python tools/micro/st_probe_levels.py $v; done > gpurun_out/r02q_levels.txt 2>&1; echo "levels $?"
timeout 600 python tools/micro/st_timing.py > gpurun_out/r02q_timing.txt 2>&1; echo "timing $?"
