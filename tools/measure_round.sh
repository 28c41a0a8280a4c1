#!/bin/bash
# usage: tools/measure_round.sh TAG -- the evidence set of one build on one box (run under gpurun):
# bench line (default bench.py), the ncu launch list of the bench step, one ncu --set full capture of
# the headline solve_to_kernel launch and of the persistent IK solver, their summaries, the per-pipe
# roofline JSON and the DRAM bytes of the headline launch.  Outputs under gpurun_out/TAG_*.
T=$1; O=gpurun_out
timeout 900 python bench.py > $O/${T}_bench.log 2>&1; tail -1 $O/${T}_bench.log > $O/${T}_bench.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"solve_to_kernel|select_kernel|ik_persist_init_kernel" -c 30 --csv --log-file $O/${T}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline --no-e2e > $O/${T}_launches.log 2>&1
bash tools/prof.sh ${T}_to
python tools/ncu_summary.py $O/${T}_to.ncu-rep > $O/${T}_to_summary.txt 2>&1
python tools/pipes_from_ncu.py $O/${T}_to.ncu-rep $O/${T}_pipes.json solve_to_kernel > $O/${T}_pipes.log 2>&1
ncu -i $O/${T}_to.ncu-rep --page source --csv --print-source cuda,sass > $O/${T}_to_src.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:solve_ik_kernel -c 1 -o $O/${T}_ik \
  python tools/prof_ik.py 1000 0 1 > $O/${T}_ik.log 2>&1
python tools/ncu_summary.py $O/${T}_ik.ncu-rep > $O/${T}_ik_summary.txt 2>&1
ncu -i $O/${T}_to.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum > $O/${T}_to_dram.csv 2>&1
rm -f $O/${T}_ik.ncu-rep
# config-5 slice of the large-world build (application replay: an earlier build did not launch under kernel replay)
timeout 1200 ncu --replay-mode application --set full --clock-control none --import-source on -k regex:solve_to_kernel -c 1 \
  -o $O/${T}_c5 python tools/prof_cfg5.py 64 10 > $O/${T}_c5.log 2>&1
python tools/ncu_summary.py $O/${T}_c5.ncu-rep > $O/${T}_c5_summary.txt 2>&1
ncu -i $O/${T}_c5.ncu-rep --page source --csv --print-source cuda,sass > $O/${T}_c5_src.csv 2>/dev/null
rm -f $O/${T}_c5.ncu-rep
