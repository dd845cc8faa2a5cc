#!/bin/bash
# Box SpMV launch-shape sweep (the fast MPK step of the PZ schedule, separable
# plane sums): default library vs the variant builds in lib/var/ (CS_DEFINES).
#   gpurun -- bash tools/box_sweep.sh > gpurun_out/box_sweep.txt
for n in 256 512; do
  CS_BENCH_NOP=1 python tools/spmv_micro.py --n $n --kinds mpk_fast --reps 50 2>&1 | tail -1
  CS_BENCH_NOP=1 CS_BOX_SEP=0 python tools/spmv_micro.py --n $n --kinds mpk_fast --reps 50 2>&1 | tail -1 | sed 's/^/sep=0 /'
  for lib in paper_2603_09790_b200/lib/var/*.so; do
    CS_BENCH_NOP=1 CS_LIB=$lib python tools/spmv_micro.py --n $n --kinds mpk_fast --reps 50 2>&1 | tail -1
  done
done
