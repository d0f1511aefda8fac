# usage: bash ab_cmd.sh TAG BASE_LIB
T=$1; B=$2
for i in 1 2 3; do
 MWT_LIB_PATH=$B python bench.py --no-extra --no-e2e --no-cpu --steps 50 | python -c 'import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print("base",d["value"],d["roofline"]["kernel_ms"])' >> gpurun_out/ab_$T.txt 2>&1
 python bench.py --no-extra --no-e2e --no-cpu --steps 50 | python -c 'import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print("new ",d["value"],d["roofline"]["kernel_ms"])' >> gpurun_out/ab_$T.txt 2>&1
done
MWT_LIB_PATH=$B python tools/ab_variants.py 22 2 >> gpurun_out/ab_$T.txt 2>&1
python tools/ab_variants.py 22 2 >> gpurun_out/ab_$T.txt 2>&1
