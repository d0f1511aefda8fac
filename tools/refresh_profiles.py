import json, shutil, subprocess, sys
tag=sys.argv[1]
line=open(f'gpurun_out/bench_{tag}.json').read().strip().splitlines()[-1]
d=json.loads(line)
print('value',d['value'],'ms',d['ms_per_step'],'frac',d['roofline']['frac'],d['roofline']['kernel_ms'],'e2e',d['e2e']['value'],'cpu',d['cpu_baseline']['value'], d['clocks'])
open('profiles/r01_bench.json','w').write(line+'\n')
ref=open(f'gpurun_out/bench_ref_{tag}.json').read().strip().splitlines()[-1]
open('profiles/r01_bench_reference.json','w').write(ref+'\n')
shutil.copy(f'gpurun_out/launches_{tag}.csv','profiles/r01_launches.csv')
steps=int(d['roofline']['algo_bytes_per_launch']//32)
st=subprocess.run(['python','tools/ncu_stats.py',f'gpurun_out/prof_{tag}.ncu-rep','16777216',str(steps)],capture_output=True,text=True).stdout
open('profiles/r01_ncu_stats.json','w').write(st)
s=subprocess.run(['python','tools/ncu_summary.py',f'gpurun_out/prof_{tag}.ncu-rep'],capture_output=True,text=True).stdout
t=subprocess.run(['python','tools/ncu_src.py',f'gpurun_out/prof_{tag}.ncu-rep','k_trace','25'],capture_output=True,text=True).stdout
hdr=("ncu --set full --import-source on --clock-control none -k regex:k_trace -s 2 -c 1 "
     "python bench.py --profile --steps 1 --warmup 3   (B200, round 1; box-entry launch, 2^24 rays, "
     "Lines-1024 MWT; walk table, boundary table and segments staged in shared memory by cp.async.bulk)\n"
     "summaries: tools/ncu_summary.py (metrics, opcode mix), tools/ncu_src.py (per source function / line), "
     "tools/ncu_stats.py -> r01_ncu_stats.json\n\n")
open('profiles/r01_ncu_k_trace.txt','w').write(hdr+s+"\n\n"+t)
sj=json.loads(st)
tr={"_note":"dram__bytes_read.sum + dram__bytes_write.sum of the dominant kernel (box-entry k_trace launch, 2^24 rays), one ncu --set full capture per round; see profiles/rNN_ncu_k_trace.txt",
    "lines1024/mwt":{"round":1,"dram_bytes_per_launch":int(sj['dram_bytes']),"report":"profiles/r01_ncu_k_trace.txt"}}
json.dump(tr,open('profiles/traffic.json','w'),indent=1)
print(json.dumps({k:sj[k] for k in ('duration_ms','warp_instructions_per_ray','warp_instructions_per_step','issue_active_pct','branch_efficiency_pct','achieved_occupancy_pct')}))
print('per_config', {k: round(v['rays_per_s']/1e9,2) for k,v in d['per_config'].items()})
print('lfl', {k: round(v['rays_per_s']/1e9,2) for k,v in d['like_for_like'].items() if isinstance(v, dict)})
print('achieved', d['roofline']['achieved'])
