#!/bin/bash
# Round artefacts on one B200: bench line, launch list, full ncu capture of the sweep.
set -u
python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; tail -c 2000 gpurun_out/bench.json
python bench.py --steps 20 --warmup 3 --precision fp32 --no-cpu-baseline > gpurun_out/bench_fp32.json 2>&1
python bench.py --steps 20 --warmup 3 --precision mixed --no-cpu-baseline > gpurun_out/bench_mixed.json 2>&1
python scripts/profile_frame.py --frames 2 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches.csv python scripts/profile_frame.py --frames 2 > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:oras_sweep -s 4 -c 1 \
    -o gpurun_out/sweep_full python scripts/profile_frame.py --frames 2 > gpurun_out/ncu_full.log 2>&1
echo done
