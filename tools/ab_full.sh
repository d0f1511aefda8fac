# usage: bash tools/ab_full.sh TAG BASE_LIB -- bench lines (value, like-for-like) base vs new
T=$1; B=$2
X='import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);l=d["like_for_like"];print(d["value"],d["roofline"]["kernel_ms"],{k:round(v["rays_per_s"]/1e9,3) for k,v in l.items() if isinstance(v,dict)})'
for i in 1 2; do
 echo -n "base " >> gpurun_out/ab_$T.txt; MWT_LIB_PATH=$B python bench.py --no-e2e --no-cpu --steps 30 | python -c "$X" >> gpurun_out/ab_$T.txt 2>&1
 echo -n "new  " >> gpurun_out/ab_$T.txt; python bench.py --no-e2e --no-cpu --steps 30 | python -c "$X" >> gpurun_out/ab_$T.txt 2>&1
done
