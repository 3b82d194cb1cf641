#!/bin/bash
# bench.py (no CPU baseline) on the default library and on compile-time
# variants variants/libhz_<name>.so (scripts/build_variant.py), interleaved:
#   bash scripts/bench_variants.sh name1 name2 ...   -> gpurun_out/bench_variants.jsonl
cd "$(dirname "$0")/.."
out=gpurun_out/bench_variants.jsonl
: > $out
for rep in 1 2; do
  for v in default "$@"; do
    if [ "$v" = default ]; then unset HZ_LIB_PATH; else export HZ_LIB_PATH=$PWD/variants/libhz_$v.so; fi
    line=$(timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>>gpurun_out/bench_variants.err | tail -1)
    python - "$v" "$line" >> $out <<'PY'
import json, sys
d = json.loads(sys.argv[2])
k = d["kernels"]
print(json.dumps({"variant": sys.argv[1], "value": round(d["value"], 2), "sm_mhz": d["clocks"]["sm_mhz"],
                  "L1_sweep_us": k.get("jacobi_stencil_c64_L1", {}).get("avg_us"),
                  "gram_us": k.get("multi_gram_c128", {}).get("avg_us")}))
PY
  done
done
cat $out
