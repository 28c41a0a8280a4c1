#!/bin/bash
# usage: tools/prof.sh NAME [PROBLEMS=64] [ITERS=100] -- ncu --set full of the first solve_to_kernel launch of
# bench.py at the bench configuration (64 problems: the sequential kernel, ~4.3 waves at 2 CTAs/SM)
P=${2:-64}; IT=${3:-100}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:solve_to_kernel -c 1 -o gpurun_out/$1 \
  python bench.py --steps 1 --warmup 0 --problems $P --iters $IT --no-cpu-baseline --no-e2e --no-extras > gpurun_out/$1.log 2>&1
tail -2 gpurun_out/$1.log
