#!/bin/bash
# A/B of library builds on the bench (interleaved, 2 rounds).
# usage: bash tools/ab_run.sh TAG "bench args" lib1 lib2 ...
# appends "<lib> <args> rays/s(1e9) kernel_ms" lines to gpurun_out/ab_TAG.txt
T=$1; A=$2; shift 2
X='import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(round(d["value"]/1e9,3),round(d["roofline"]["kernel_ms"],4))'
for i in 1 2; do
 for L in "$@"; do
  echo -n "$L $A " >> gpurun_out/ab_$T.txt
  MWT_LIB_PATH=$L python bench.py --no-extra --no-e2e --no-cpu --steps 30 $A | python -c "$X" >> gpurun_out/ab_$T.txt 2>&1
 done
done
