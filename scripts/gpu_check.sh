#!/bin/bash
# GPU smoke of a change: parity suite summary + per-kernel device times.
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest-gpu: $(tail -1 gpurun_out/pytest_gpu.log)"
grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head -5
python scripts/quick_perf.py 2>&1 | grep -A1 "^C3"
