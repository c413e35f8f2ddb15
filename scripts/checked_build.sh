#!/bin/bash
# The checked build: the same sources with -DSEG_DEBUG (device-side SEG_DCHECK bounds checks on every
# shared-memory queue, ring stage, tile index and scatter position; a violation traps), then the GPU
# parity suite and the full-size bench configuration against it.  Stand-in for compute-sanitizer,
# which the GPU pool does not offer.  Usage (GPU box): bash scripts/checked_build.sh
set -u
cd "$(dirname "$0")/.."
mkdir -p build/checked gpurun_out
python - <<'PY'
import subprocess
from paper_1912_11494_b200 import _build
subprocess.check_call([_build.nvcc(), *_build.NVCC_FLAGS, "-DSEG_DEBUG", "-o", "build/checked/libsegb200.so",
                       *_build.SOURCES])
print("checked build ok")
PY
export SEG_LIB=$PWD/build/checked/libsegb200.so
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
echo "checked pytest rc=${PIPESTATUS[0]}"
timeout 300 python bench.py --steps 3 --warmup 3 2>&1 | tail -1 | cut -c1-200
echo "checked bench rc=${PIPESTATUS[0]}"
