#!/usr/bin/env bash
# Temporal-blocking kernel variants: build here (MODE=build), time on a B200 via gpurun
# (MODE=run).  Each variant recompiles the f64 and f32-native units with extra -D flags and
# links them with the product objects into build/tune/<name>/libps.so, selected at run
# time with PS_LIBRARY; the product build is untouched.
#
# Round-1 history (C4 f64 P9 T=4, 40 steps): base 475, minb2 477, rb6 475 GLUP/s; 11 consumer
# warps in one block (164 registers, no spills) 513-520; a variant starting the accumulator at the first product (one DADD fewer, -0.0
# fixed up on the integer pipe) ran 460; a skewed stage pipeline (stage t lagging R+1 rows so
# the TS stages of a step are independent: 4x the add chains per warp, bitwise correct) needs
# ~200 registers and ran 452 (7 warps) / 430 (11 warps, spills).  Register caps: a 9-warp block can use at most
# 168 registers per thread (3 warps share one SM sub-partition's 16K registers).
# Session 4: two 16-B vectors per lane in 7 consumer warps (PS_TB_VM=2, 8 warps -> 228
# registers, no spills): C4 535 -> 558-585; with it, starting the sum at the first product
# and fixing -0.0 on p0 only (off the add chain) still lost (540); f32 P13 T=4 with two
# vectors per lane: 718 (narrow windows) / 634 (wide) vs 1009 -- f32 and P13 keep one vector.
# The producer warp leaves one SM sub-partition with a consumer warp fewer; removing it
# lost both ways: folded into consumer warp 0 (C4 528, C5 801) and as warp-private
# pipelines, each warp issuing its own copies into its own ring (C4 524, C5 720, C3 274).
# What worked: warpgroup specialisation (setmaxnreg): warpgroup 0 shrinks to 40/32
# registers and its warp 0 produces, 8 (two-vector) or 12 (f32) consumer warps grow to
# 232/160 -- every sub-partition gets the same number of consumers: C4 579-600 -> 616-625,
# C5 1036 -> 1052, C3 f32 804 -> 826 (P13 f64 flat, periodic C2 291 vs 321: not used there).
# Session 5: 6 rows per pipeline slot for radius 2 (PS_TB_RB=6): C5 1052 -> 1080, C3 f32
# 827 -> 837 (8 and 10 rows exceed shared memory; radius 1 keeps 3: 6 rows do not fit
# the two-vector f64 ring); 4 ring stages (PS_TB_NS=4): flat; f64 narrow windows: C3 T=4
# 319 vs 358 at T=2, C2 323 vs 342.  6 rows for radius 1 (periodic C2: 317 vs 333) and 6 rows
# in 2 ring stages (C4 584 vs 586-634, C2 324, C5 1038 vs 1079): dropped.
# Radius-2 f32 ring shape at ~equal shared memory (C5 / C3 f32): 6x3 rows 1079 / 840,
# 4x5 995 / 781, 3x6 938 / 748, 8x2 1076 / 830, 9x2 1078 / 821 -- rows per slot matter
# (per-slot barrier overhead), ring depth beyond 2 slots of slack does not.
set -e
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
NV="nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Iinclude"
CSRC=paper_1904_04048_b200/csrc
declare -A VARIANTS=(
  [cur]=""

)
if [ "${MODE:-build}" = build ]; then
  make -s -j4 paper_1904_04048_b200/libps.so
  for v in "${!VARIANTS[@]}"; do
    (mkdir -p build/tune/$v &&
     $NV ${VARIANTS[$v]} -c -o build/tune/$v/ps_kern_f64.o $CSRC/ps_kern_f64.cu &&
     $NV ${VARIANTS[$v]} -c -o build/tune/$v/ps_kern_f32n.o $CSRC/ps_kern_f32n.cu &&
     $NV -shared -o build/tune/$v/libps.so build/obj/ps_device.o build/tune/$v/ps_kern_f64.o \
       build/obj/ps_kern_f32r.o build/tune/$v/ps_kern_f32n.o) &
  done
  wait
else
  mkdir -p gpurun_out
  for rep in ${REPS:-1 2}; do
  for v in "${!VARIANTS[@]}"; do
    for ct in ${CONFIGS:-C4:4 C5:4 C2:4 C3:2 C3f32:4}; do
      c=${ct%%:*}; t=${ct##*:}
      PS_LIBRARY="build/tune/$v/libps.so" timeout 200 python bench.py --config $c --steps ${STEPS:-40} \
        --no-e2e --no-cpu --tsteps $t > "gpurun_out/tbv_${v}_${c}_$rep.log" 2>&1 || true
    done
  done
  done
fi
