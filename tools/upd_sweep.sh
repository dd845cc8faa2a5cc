#!/bin/bash
# Update / pack pass A/B (PZ schedule): default vs variant builds in lib/var/.
for n in 256 512; do
  CS_BENCH_PZ=1 python tools/spmv_micro.py --n $n --kinds pack8,update8 --reps 30 2>&1 | tail -1
  for lib in paper_2603_09790_b200/lib/var/*.so; do
    CS_BENCH_PZ=1 CS_LIB=$lib python tools/spmv_micro.py --n $n --kinds pack8,update8 --reps 30 2>&1 | tail -1
  done
  python tools/spmv_micro.py --n $n --kinds pack8,update8 --reps 30 2>&1 | tail -1 | sed 's/^/storedP /'
done
