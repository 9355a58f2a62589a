#!/bin/bash
# A/B timing of library variants in variants/*.so (dev aid); extra env per run via AB_ENVS
for v in variants/*.so; do
  for envs in ${AB_ENVS:-NONE=1}; do
    echo "== $v $envs"
    env $envs GRSOLVE_LIB=$PWD/$v timeout 300 python scripts/time_configs.py ${@:-c2 c3 c4} 2>&1 | grep -v "^c2 greedy"
  done
done
