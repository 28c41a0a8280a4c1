#!/bin/bash
# usage: tools/ab2.sh "v1 v2 ..." [rounds=2] -- cfg2 bench (10 steps) and cfg3 IK (1000 goals, 7 reps) per variant,
# interleaved over rounds (drift between variants shows up as round-to-round spread)
R=${2:-2}
for r in $(seq 1 $R); do for v in $1; do
  CRB_LIB=tools/libcrb_$v.so timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-extras --steps 10 2>&1 | tail -1 | \
  python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg2', round(d['value']/1e6,1), 'M evals/s', round(d['ms_per_step'],2), 'ms', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"
  CRB_LIB=tools/libcrb_$v.so timeout 300 python tools/prof_ik.py 1000 0 7 2>&1 | tail -1
done; done
