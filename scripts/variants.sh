#!/bin/bash
# Sweep-kernel variants (warps per CTA) on the 4K frame, device-resident.
for v in "SI_SWEEP_WARPS64=4" "SI_SWEEP_WARPS64=2"; do
  echo "== $v"; env $v python scripts/quick_perf.py 2>&1 | grep -A1 "C3 FP64"
done
for v in "SI_SWEEP_WARPS32=1" "SI_SWEEP_WARPS32=2" "SI_SWEEP_WARPS32=4"; do
  echo "== $v"; env $v python scripts/quick_perf.py 2>&1 | grep -A1 "C3 FP32"
done
