# build A/B library variants here (cross-compiled, in parallel) into abl/NAME.so for scripts/ab_build.py "lib:abl/NAME.so"
# usage: scripts/ab_prebuild.sh NAME1 "-DX=1" NAME2 "-DY=1 -DZ=2" ...
set -e
cd "$(dirname "$0")/.."
mkdir -p abl
SRC="paper_1912_11494_b200/csrc/seg_api.cu paper_1912_11494_b200/csrc/classify.cu paper_1912_11494_b200/csrc/group.cu paper_1912_11494_b200/csrc/resample.cu"
while [ $# -ge 2 ]; do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -shared -Xcompiler -fPIC -Iinclude $2 -o abl/$1.so $SRC &
  shift 2
done
wait
ls -la abl/
