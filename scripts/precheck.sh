#!/bin/bash
# Build + CPU test tier; run before every gpurun call.
set -e
cd "$(dirname "$0")/.."
python paper_1607_00968_b200/build_ext.py > /dev/null
timeout 900 python -m pytest tests -x -q -m "not gpu" 2>&1 | tail -2
