#!/bin/bash
# Register / spill summary of one CUDA source (development tool): tools/ptxas_regs.sh FILE.cu [grep-pattern]
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -Xptxas=-v \
  -I "$(dirname "$0")/../include" -c -o /tmp/_ptxas_regs.o "$1" 2>&1 |
  awk '/Compiling entry function/ {f=$0; sub(/.*function ./,"",f); sub(/. for .*/,"",f)}
       /spill stores/ {sp=$0; sub(/.*ptxas info *: */,"",sp)}
       /Used [0-9]+ registers/ {r=$0; sub(/.*Used /,"",r); sub(/ registers.*/,"",r); print r, sp, f}' |
  grep -E "${2:-.}"
