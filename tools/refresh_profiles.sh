#!/bin/bash
# Refresh the committed ncu evidence (run on the GPU box from the repo root): launch list of
# the bench command, --set full tables of one animation frame and of the SPEC train step,
# per-launch DRAM traffic, SASS evidence. Each profiled command first runs without ncu.
# Usage: bash tools/refresh_profiles.sh [round tag, default r2]
set -o pipefail
R=${1:-r2}
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/rp_bench.json 2> gpurun_out/rp_bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_$R.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/rp_ncu1.log 2>&1 || exit 2
python tools/prof_frame.py 1 tcgen05 > /dev/null || exit 3
rm -f /tmp/frame.ncu-rep /tmp/train.ncu-rep
ncu --set full --import-source on --clock-control none -o /tmp/frame python tools/prof_frame.py 1 tcgen05 \
  > gpurun_out/rp_ncu2.log 2>&1 || exit 4
python tools/ncu_summary.py /tmp/frame.ncu-rep gpurun_out/ncu_${R}_frame.json > /dev/null || exit 5
python tools/ncu_table.py gpurun_out/ncu_${R}_frame_kernels.md /tmp/frame.ncu-rep || exit 6
python tools/ncu_traffic.py gpurun_out/ncu_${R}_frame.json gpurun_out/ncu_traffic.json || exit 7
python tools/prof_train.py 2 > /dev/null || exit 8
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${R}_train.csv \
  python tools/prof_train.py 6 > gpurun_out/rp_ncu3.log 2>&1 || exit 9
python tools/launch_table.py gpurun_out/launches_${R}_train.csv 150 > gpurun_out/launches_${R}_train.md || exit 10
ncu --set full --clock-control none -k regex:"newton|field_team|field_bwd|grid_scatter|composite|adam|march|weights|finalize|owner|density" \
  -c 40 -o /tmp/train python tools/prof_train.py 2 > gpurun_out/rp_ncu4.log 2>&1 || exit 11
python tools/ncu_table.py gpurun_out/ncu_${R}_train_kernels.md /tmp/train.ncu-rep || exit 12
cp /tmp/frame.ncu-rep gpurun_out/frame_$R.ncu-rep
echo done
