#!/bin/bash
# Round-2 (session 3) evidence in one GPU call: GPU tests, smoke, the bench line + reference arm,
# other configs, the launch list, level-step DRAM traffic and ncu --set full of level_update6.
mkdir -p gpurun_out
T=${TAG:-s3z}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${T}_pytest.log
cp gpurun_out/parity_errors.json gpurun_out/${T}_parity_errors.json 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"; cat gpurun_out/${T}_bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_ref.json 2>&1; tail -1 gpurun_out/${T}_bench_ref.json
timeout 1200 python tools/bench_configs.py cfg1 cfg4 cfg4g cfg5 > gpurun_out/${T}_configs.jsonl 2>&1; cat gpurun_out/${T}_configs.jsonl | cut -c1-200
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python tools/profile_once.py > /dev/null 2>&1
python tools/launch_list.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launch_list.txt 2>&1
python tools/launch_summary.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launch_summary.txt 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:level_update --csv --log-file gpurun_out/${T}_level_traffic.csv python tools/profile_once.py > /dev/null 2>&1
python tools/traffic_json.py gpurun_out/${T}_level_traffic.csv 13 > gpurun_out/${T}_traffic.json 2>&1
for spec in "13:0" "12:2" "7:9"; do
  lv=${spec%%:*}; skip=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:level_update --launch-skip $skip -c 1 -o gpurun_out/${T}_level_l${lv} -f python tools/profile_once.py > /dev/null 2>&1
done
python tools/ncu_summary.py gpurun_out/${T}_level_l13.ncu-rep gpurun_out/${T}_level_l12.ncu-rep gpurun_out/${T}_level_l7.ncu-rep > gpurun_out/${T}_ncu_summary.txt 2>&1
echo done
