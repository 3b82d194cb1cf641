#!/bin/bash
# Per-kernel event profile of one 8-column bench block (profile_solve.py 8 c64 60)
# for the default library and each variants/libhz_<name>.so given.
# Usage (GPU box): bash scripts/lib_ab.sh name1 name2 ... [| grep pattern]
echo "== default"
python scripts/profile_solve.py 8 c64 60 2>&1 | head -9
for v in "$@"; do
  echo "== variant $v"
  HZ_LIB_PATH=variants/libhz_$v.so python scripts/profile_solve.py 8 c64 60 2>&1 | head -9
done
