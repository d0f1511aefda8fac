# usage: bash tools/ab_libs.sh TAG lib1 lib2 ... -- headline bench value per library, interleaved, 2 rounds
T=$1; shift
X='import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(round(d["value"]/1e9,3),round(d["roofline"]["kernel_ms"],4))'
for i in 1 2; do
 for L in "$@"; do
  echo -n "$L " >> gpurun_out/ab_$T.txt; MWT_LIB_PATH=$L python bench.py --no-extra --no-e2e --no-cpu --steps 50 | python -c "$X" >> gpurun_out/ab_$T.txt 2>&1
 done
done
