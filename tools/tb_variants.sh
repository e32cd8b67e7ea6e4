#!/usr/bin/env bash
# Temporal-blocking kernel variants for the f64 unit: build here (MODE=build), time on a
# B200 via gpurun (MODE=run).  Round-1 result (C4 f64 P9 T=4, 40 steps): base 475,
# minb2 477, rb6 475 GLUP/s; a variant starting the accumulator at the first product (one
# DADD fewer, -0.0 fixed up on the integer pipe) ran 460 — the kernel sits on a plateau.  Each variant recompiles ps_kern_f64.cu with extra -D flags
# and links it with the product objects into build/tune/<name>/libps.so, selected at run
# time with PS_LIBRARY; the product build is untouched.
set -e
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
NV="nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Iinclude"
CSRC=paper_1904_04048_b200/csrc
declare -A VARIANTS=(
  [base]=""
  [minb2]="-DPS_TB_MINB=2"
  [rb6]="-DPS_TB_RB=6"
)
if [ "${MODE:-build}" = build ]; then
  make -s -j4 paper_1904_04048_b200/libps.so
  for v in "${!VARIANTS[@]}"; do
    (mkdir -p build/tune/$v && $NV ${VARIANTS[$v]} -c -o build/tune/$v/ps_kern_f64.o $CSRC/ps_kern_f64.cu &&
     $NV -shared -o build/tune/$v/libps.so build/obj/ps_device.o build/tune/$v/ps_kern_f64.o \
       build/obj/ps_kern_f32r.o build/obj/ps_kern_f32n.o) &
  done
  wait
else
  mkdir -p gpurun_out
  for rep in 1 2; do
  for v in "${!VARIANTS[@]}"; do
    for c in ${CONFIGS:-C4 C3}; do
      PS_LIBRARY="build/tune/$v/libps.so" timeout 200 python bench.py --config $c --steps ${STEPS:-40} \
        --no-e2e --no-cpu --tsteps ${TS:-4} > "gpurun_out/tbv_${v}_${c}_$rep.log" 2>&1 || true
    done
  done
  done
fi
