set -x
timeout 600 python tools/level_breakdown.py C2b 2>&1 | tail -40
