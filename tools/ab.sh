#!/bin/bash
# usage: tools/ab.sh "v1 v2 ..." "P1 P2 ..." [extra bench args] -- bench.py with CRB_LIB=tools/libcrb_$v.so
for P in $2; do for v in $1; do
  CRB_LIB=tools/libcrb_$v.so timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-extras --problems $P --steps 10 $3 2>&1 | tail -1 | \
  python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['clocks']; print('$v P=$P', round(d['value']/1e6,1), 'M evals/s', round(d['ms_per_step'],2), 'ms', c.get('sm_mhz'), c.get('sm_min_mhz'), c.get('samples'), c.get('reasons'))"
done; done
