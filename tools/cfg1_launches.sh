#!/bin/bash
# launch list of one cfg1-shaped (N=2^14, m=64, r=32) factorize + solve
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg1_launches.csv python tools/profile_once.py 16384 32 > /dev/null 2>&1
python tools/launch_list.py gpurun_out/cfg1_launches.csv > gpurun_out/cfg1_launch_list.txt 2>&1
n=$(wc -l < gpurun_out/cfg1_launch_list.txt); tail -n $((n/2)) gpurun_out/cfg1_launch_list.txt
