#!/bin/bash
# Refresh the committed ncu evidence (run on the GPU box from the repo root):
# launch list of the bench command, --set full tables of one animation frame and of the
# SPEC train step, per-launch DRAM traffic. Each profiled command first runs without ncu.
set -o pipefail
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/rp_bench.json 2> gpurun_out/rp_bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/rp_ncu1.log 2>&1 || exit 2
python tools/prof_frame.py 1 tcgen05 > /dev/null || exit 3
rm -f /tmp/frame.ncu-rep /tmp/train.ncu-rep
ncu --set full --import-source on --clock-control none -o /tmp/frame python tools/prof_frame.py 1 tcgen05 \
  > gpurun_out/rp_ncu2.log 2>&1 || exit 4
python tools/ncu_summary.py /tmp/frame.ncu-rep gpurun_out/ncu_frame.json > /dev/null || exit 5
python tools/ncu_table.py gpurun_out/ncu_frame_kernels.md /tmp/frame.ncu-rep || exit 6
python tools/ncu_traffic.py gpurun_out/ncu_frame.json gpurun_out/ncu_traffic.json || exit 7
python tools/prof_train.py 2 > /dev/null || exit 8
ncu --set full --clock-control none -k regex:"newton|field_team|field_bwd|grid_scatter|composite|adam|march|weights|finalize|owner|density" \
  -c 40 -o /tmp/train python tools/prof_train.py 2 > gpurun_out/rp_ncu3.log 2>&1 || exit 9
python tools/ncu_table.py gpurun_out/ncu_train_kernels.md /tmp/train.ncu-rep || exit 10
echo done
