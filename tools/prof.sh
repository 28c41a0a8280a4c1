#!/bin/bash
# usage: tools_prof.sh NAME  -- ncu full capture of solve_to_kernel on a 1-wave problem set
timeout 600 ncu --set full --clock-control none --import-source on -k regex:solve_to -c 1 -o gpurun_out/$1 python bench.py --steps 1 --warmup 0 --problems 9 --iters 20 --no-cpu-baseline --no-e2e > gpurun_out/$1.log 2>&1
tail -2 gpurun_out/$1.log
