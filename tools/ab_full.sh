#!/bin/bash
# usage: tools/ab_full.sh "v1 v2 ..." -- full bench (with extras) per variant, key numbers only
for v in $1; do
  CRB_LIB=tools/libcrb_$v.so timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 2>&1 | tail -1 | \
  python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['extras']; print('$v', 'cfg2', round(d['value']/1e6,1), 'ik/s', round(e['cfg3_ik']['ik_queries_per_s']), 'ik+f1', round(e['cfg3_ik']['with_particles']['ik_queries_per_s']), 'f1TO ms', round(e['f1_particle_to']['ms_particle_plus_lbfgs'],1), 'cfg4', round(e['cfg4_batched_to']['problems_per_s']), 'cfg5', round(e['cfg5_dense']['evals_per_s']/1e6,2), 'f2', round(e['f2_motion_gen']['P64']['ms_per_batch'],1))"
done
