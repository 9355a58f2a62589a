#!/bin/bash
# build variants/libgr_a_head.so from HEAD and variants/libgr_b_work.so from the
# working tree (dev aid for A/B timing with scripts/ab.sh)
set -e
mkdir -p variants
rm -f variants/*.so
F="-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -shared -Iinclude"
T=$(mktemp -d)
git archive HEAD paper_2011_08373_b200/csrc include | tar -x -C $T
/usr/local/cuda/bin/nvcc $F -I$T/include -o variants/libgr_a_head.so $T/paper_2011_08373_b200/csrc/*.cu &
/usr/local/cuda/bin/nvcc $F -o variants/libgr_b_work.so paper_2011_08373_b200/csrc/*.cu &
wait
rm -rf $T
cp variants/libgr_b_work.so paper_2011_08373_b200/libgrsolve.so
