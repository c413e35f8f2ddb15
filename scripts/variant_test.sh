#!/bin/bash
# Build the library with extra nvcc defines into build/variant/ and run the GPU parity suite against it
# (SEG_LIB).  Usage (GPU box): bash scripts/variant_test.sh "-DSEG_TC" [pytest -k expr]
set -u
cd "$(dirname "$0")/.."
mkdir -p build/variant gpurun_out
DEFS="$1"
python - "$DEFS" <<'PY'
import subprocess, sys
from paper_1912_11494_b200 import _build
subprocess.check_call([_build.nvcc(), *_build.NVCC_FLAGS, *sys.argv[1].split(), "-o", "build/variant/libsegb200.so",
                       *_build.SOURCES], stderr=subprocess.DEVNULL)
print("variant build ok:", sys.argv[1])
PY
export SEG_LIB=$PWD/build/variant/libsegb200.so
timeout 1500 python -m pytest tests -m gpu -x -q ${2:+-k "$2"} 2>&1 | tail -15
echo "variant pytest rc=${PIPESTATUS[0]}"
