#!/bin/bash
# Round-end evidence run on ONE GPU box (dev aid).  Every ncu pass runs only
# after the same command exited 0 without ncu.  Outputs: gpurun_out/<R>/.
#   tests.log           pytest -m gpu
#   bench.json          python bench.py (all configs: the driver's command)
#   bench_reference.json  python bench.py --impl reference
#   launches_c2.csv     ncu launch list of the C2 bench command (cold, serialised: shares only)
#   q_c2/q_c3/q_c4.ncu-rep  ncu --set full of queue_kernel (the timed fused / weighted walks)
#   count_c5.ncu-rep    ncu --set full of count_kernel (C5 recount pass)
#   lscatter_c5 / lgreedy_c5.ncu-rep  the list greedy (f3) kernels
#   onegpu/             bench.py N = 2 on one GPU (gloo; functional only)
R=${1:-r02}
O=gpurun_out/$R
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.log
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
B="python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
if timeout 600 $B > $O/launch_run.json 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_c2.csv $B > $O/ncu_launch.log 2>&1
fi
for c in c2 c3 c4; do
  if timeout 300 python scripts/prof_c2.py $c > $O/prof_$c.log 2>&1; then
    timeout 900 ncu --set full --import-source on --clock-control none -k regex:queue_kernel \
      --launch-count 1 -o $O/q_$c python scripts/prof_c2.py $c > $O/ncu_q_$c.log 2>&1
  fi
done
if timeout 600 python scripts/prof_c5.py --full > $O/prof_c5.log 2>&1; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:count_kernel \
    --launch-skip 4 --launch-count 1 -o $O/count_c5 python scripts/prof_c5.py --full > $O/ncu_count.log 2>&1
fi
if timeout 300 python scripts/time_lists.py > $O/time_lists.log 2>&1; then
  for k in lscatter lgreedy; do
    timeout 900 ncu --set full --import-source on --clock-control none -k regex:${k}_kernel \
      --launch-skip 2 --launch-count 1 -o $O/${k}_c5 python scripts/time_lists.py > $O/ncu_$k.log 2>&1
  done
fi
bash scripts/onegpu_multirank.sh $O/onegpu
ls -la $O
