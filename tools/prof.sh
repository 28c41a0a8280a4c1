#!/bin/bash
# usage: tools/prof.sh NAME [PROBLEMS] [ITERS] -- ncu --set full of solve_to_kernel (~1 wave at 2 CTAs/SM)
P=${2:-10}; IT=${3:-100}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:solve_to -c 1 -o gpurun_out/$1 \
  python bench.py --steps 1 --warmup 0 --problems $P --iters $IT --no-cpu-baseline --no-e2e > gpurun_out/$1.log 2>&1
tail -2 gpurun_out/$1.log
