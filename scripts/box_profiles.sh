#!/bin/bash
# Round-end evidence run on the GPU box (dev aid): bench lines of every
# config, the ncu launch list of the default bench command, and one
# ncu --set full capture of the top kernel (each ncu pass only after its
# command exited 0 without ncu).  Outputs land in gpurun_out/prof/.
R=${1:-r01}
O=gpurun_out/prof
mkdir -p $O
for c in c2 c3 c4 c5; do
  timeout 900 python bench.py --config $c > $O/${R}_bench_$c.json 2> $O/${R}_bench_$c.err || echo "bench $c failed"
done
timeout 900 python bench.py --impl reference > $O/${R}_bench_reference.json 2> $O/${R}_bench_reference.err
timeout 900 python bench.py --impl reference --config c5 > $O/${R}_bench_reference_c5.json 2>> $O/${R}_bench_reference.err
# launch list of the bench command (cold-cache, serialised: shares only)
if timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/launch_run.json 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/${R}_launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
    > $O/ncu_launch.log 2>&1
fi
# full capture of the dominant kernel at a big C2 level (PMS solve, level 16)
if timeout 300 python scripts/prof_c2.py > $O/prof_c2.log 2>&1; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:enum_kernel \
    --launch-skip 15 --launch-count 1 -o $O/${R}_enum_c2 python scripts/prof_c2.py > $O/ncu_full.log 2>&1
fi
ls -la $O
