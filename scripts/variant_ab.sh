#!/bin/bash
# A/B: default library vs variants/libhz_$1.so on the bench workload
cd "$(dirname "$0")/.."
for v in default "$@"; do
  if [ "$v" = default ]; then unset HZ_LIB_PATH; else export HZ_LIB_PATH=$PWD/variants/libhz_$v.so; fi
  echo "$v $(timeout 300 python scripts/sweep_groups.py 32,8 2>&1 | tr '\n' ' ')"
  timeout 300 python scripts/profile_solve.py 8 c64 60 2>&1 | grep -E "multi_update|multi_gram" | sed "s/^/   $v /"
done
