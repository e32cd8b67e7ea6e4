#!/usr/bin/env bash
# Build streaming / temporal-blocking kernel geometry variants into build/tune/ (run here),
# then time them on a B200 (run via gpurun with MODE=run).  Variants are selected at run
# time with PS_LIBRARY=build/tune/libps_<name>.so; the product build is untouched.
set -e
cd "$(dirname "$0")/.."
NV="nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared -Iinclude"
SRC=paper_1904_04048_b200/csrc/ps_device.cu
declare -A VARIANTS=(
  [s4x6x4]="-DPS_NW=4 -DPS_RB1=6 -DPS_RB2=5 -DPS_NS=4"
  [s8x4x3]="-DPS_NW=8 -DPS_RB1=4 -DPS_RB2=4 -DPS_NS=3"
  [s8x5x2]="-DPS_NW=8 -DPS_RB1=5 -DPS_RB2=5 -DPS_NS=2"
  [t4x3]="-DPS_TB_NW=4 -DPS_TB_NS=3"
  [t8x2]="-DPS_TB_NW=8 -DPS_TB_NS=2"
)
if [ "${MODE:-build}" = build ]; then
  mkdir -p build/tune
  for v in "${!VARIANTS[@]}"; do $NV ${VARIANTS[$v]} -o "build/tune/libps_$v.so" $SRC & done
  wait
else
  cd "${GRAFT_REPO_ROOT:-.}"
  for v in "${!VARIANTS[@]}"; do
    for c in C4 C5; do for t in 1 2 4; do
      PS_LIBRARY="build/tune/libps_$v.so" timeout 200 python bench.py --config $c --tsteps $t \
        --no-e2e --no-cpu > "gpurun_out/tune_${v}_${c}_T$t.log" 2>&1
    done; done
  done
fi
