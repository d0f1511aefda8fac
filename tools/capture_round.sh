#!/bin/bash
# One GPU call's worth of round evidence for the CURRENT build (run on the box):
#   bench lines (engine arm + reference arm), the launch list, full ncu
#   captures of the headline walk launch (FloorPlan), the Lines-1024 and
#   Hair-512 walk launches, and the kd-tree / BVH launches (FloorPlan, both
#   ray orders), written to gpurun_out/ with tag $1.
# usage: bash tools/capture_round.sh TAG [--no-tests]
T=${1:-r02}
O=gpurun_out
if [ "$2" != "--no-tests" ]; then
  python -m pytest tests -m gpu -q -rs > $O/gputest_$T.log 2>&1; echo "gputest=$?"; tail -3 $O/gputest_$T.log
fi
python bench.py > $O/bench_$T.json 2> $O/bench_$T.err; echo "bench=$?"
python bench.py --impl reference > $O/bench_ref_$T.json 2> $O/bench_ref_$T.err; echo "ref=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$T.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-extra > /dev/null 2>&1; echo "launches=$?"
NCU="ncu --set full --import-source on --clock-control none"
$NCU -k regex:k_trace -s 2 -c 1 -o $O/prof_fp_$T python bench.py --profile --steps 1 --warmup 3 > $O/ncu_fp_$T.log 2>&1; echo "fp=$?"
$NCU -k regex:k_trace -s 2 -c 1 -o $O/prof_l1k_$T python bench.py --config lines1024 --profile --steps 1 --warmup 3 > $O/ncu_l1k_$T.log 2>&1; echo "l1k=$?"
$NCU -k regex:k_trace -s 2 -c 1 -o $O/prof_hair_$T python bench.py --config hair512 --profile --steps 1 --warmup 3 > $O/ncu_hair_$T.log 2>&1; echo "hair=$?"
$NCU -k regex:"k_kd|k_bvh" -s 6 -c 2 -o $O/prof_struct_coh_$T python tools/prof_struct.py floorplan64 coherent 4194304 2 2 > $O/ncu_struct_coh_$T.log 2>&1; echo "struct_coh=$?"
$NCU -k regex:"k_kd|k_bvh" -s 6 -c 2 -o $O/prof_struct_iid_$T python tools/prof_struct.py floorplan64 iid 4194304 2 2 > $O/ncu_struct_iid_$T.log 2>&1; echo "struct_iid=$?"
$NCU -k regex:k_trace -s 2 -c 1 -o $O/prof_int_$T python tools/prof_one.py lines1024 mwt 1 4194304 6 4 > $O/ncu_int_$T.log 2>&1; echo "interior=$?"
