#!/usr/bin/env bash
# Fused-kernel tuning variants, one kernel per variant (seconds to build):
#   MODE=build bash tools/tb_tune.sh            # here: nvcc each variant's fused unit
#   gpurun -- 'MODE=run bash tools/tb_tune.sh'  # on a B200: bench each, logs in gpurun_out/
# A variant is "<name>|<config>:<T>|<unit>|<-D flags>"; its library
# build/tune/<name>/libps.so links the variant's ps_kern_<unit>_t<T>.o with the product
# objects and is selected with PS_LIBRARY.  PS_TUNE_SHAPE/PS_TUNE_TS restrict the unit to
# the one fused kernel the config runs.  ONLY="a b" selects variants.
#
# Round-2 results (40-42 steps, 1965 MHz unless noted; GLUP/s):
#   C4 (P9 f64 T=4): old (two vectors/lane, 8 WGS warps, one product per tap) 651;
#     shared products, 12 WGS warps: 4 rows x 3 slots 641, 2 x 4 543, 8 x 2 652; 11 warps +
#     producer warp (168 regs, 296 B spills) 513; two vectors per lane (644 B spills) 436.
#     200-step runs under the power cap: old 557-558 (1.68 GHz), shared 565-570 (1.57-1.62).
#   C3 (P13 f64): T=2 old 373; T=3 old, 8 WGS warps (232 regs, no spills) 381, same with
#     4-row slots 349; T=4 old 8 WGS warps 360; shared products T=2 (12 warps, 8 x 2) 336,
#     T=3 8 warps 385 (8 x 2: 358), T=3 12 warps (1 KB spills) 191.
#
# Round-2, last session (40-step runs at 1965 MHz; 200-step runs tie under the power cap):
#   C4 T=5 ring shape at equal shared memory: 8x3 752-756, 10x3 772 (now the default for
#     radius 1 where 30 rows fit), 6x4 737, 4x6 718; producer sleep 0 ns 750-756 (no change).
#   Unrolled head slots (PS_TB_SYM_HEAD): C3 T=3 451 -> 458, C4 728-758 vs 750 (noise), +7 min
#     of ptxas for the radius-2 body: off.  Producer-written slot descriptors (tile arithmetic
#     out of the consumer warps): C4 +0.5 %, C2 +2 %, C3 -9 % (spills): not kept.
#   C2 (periodic P9 T=4) after the image-loop fix: 335; shared products 258, 8 WGS warps 329.
#
# Round-1 history (tools/tb_variants.sh, now folded in here):
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
C4="-DPS_TUNE_SHAPE=ShapeP9 -DPS_TUNE_TS=4"
C3T2="-DPS_TUNE_SHAPE=ShapeP13 -DPS_TUNE_TS=2"
C3T3="-DPS_TUNE_SHAPE=ShapeP13 -DPS_TUNE_TS=3"
C3T4="-DPS_TUNE_SHAPE=ShapeP13 -DPS_TUNE_TS=4"
C2T4="-DPS_TUNE_SHAPE=ShapeP9 -DPS_TUNE_TS=4 -DPS_TUNE_BC=PS_BC_PERIODIC"
C2T5="-DPS_TUNE_SHAPE=ShapeP9 -DPS_TUNE_TS=5 -DPS_TUNE_BC=PS_BC_PERIODIC"
C5T4="-DPS_TUNE_SHAPE=ShapeP13 -DPS_TUNE_TS=4"
C4T5="-DPS_TUNE_SHAPE=ShapeP9 -DPS_TUNE_TS=5"
VARIANTS=(
  "c4t5base|C4:5|f64|$C4T5"
  "c4t5nohead|C4:5|f64|$C4T5 -DPS_TB_SYM_HEAD=0"
  "c3t3base|C3:3|f64|$C3T3"
  "c3t3nohead|C3:3|f64|$C3T3 -DPS_TB_SYM_HEAD=0"
  "c4t5_4x6|C4:5|f64|$C4T5 -DPS_TB_RB=4 -DPS_TB_NS=6"
  "c4t5_6x4|C4:5|f64|$C4T5 -DPS_TB_RB=6 -DPS_TB_NS=4"
  "c4t5_2x12|C4:5|f64|$C4T5 -DPS_TB_RB=2 -DPS_TB_NS=12"
  "c4t5_10x3|C4:5|f64|$C4T5 -DPS_TB_RB=10 -DPS_TB_NS=3"
  "c4t5_sleep0|C4:5|f64|$C4T5 -DPS_TB_PROD_SLEEP=0"
  "c4t5sleep|C4:5|f64|$C4T5 -DPS_TB_PROD_SLEEP=100"
  "c4t5sleep4|C4:5|f64|$C4T5 -DPS_TB_PROD_SLEEP=400"
  "c4t5edge|C4:5|f64|$C4T5 -DPS_TB_PROD_SLEEP=100 -DPS_TB_SYM_EDGE=1 -DPS_TB_RC_ALIGN=1"
  "c4t5align|C4:5|f64|$C4T5 -DPS_TB_PROD_SLEEP=100 -DPS_TB_RC_ALIGN=1"
  "c5sleep|C5:4|f32n|$C5T4 -DPS_TB_PROD_SLEEP=100"
  "c3t3edge|C3:3|f64|$C3T3 -DPS_TB_SYM_EDGE=2"
  "c5pair|C5:4|f32n|$C5T4 -DPS_TB_PAIR=1"
  "c5nopair|C5:4|f32n|$C5T4 -DPS_TB_PAIR=0"
  "c3t3sleep|C3:3|f64|$C3T3 -DPS_TB_PROD_SLEEP=100"
  "c3sym3a|C3:3|f64|$C3T3 -DPS_TB_SYM=2 -DPS_TB_SYM_R2_MAXT=3 -DPS_TB_WGS_NW=8 -DPS_TB_RB=8 -DPS_TB_NS=3"
  "c3sym4a|C3:4|f64|$C3T4 -DPS_TB_SYM=2 -DPS_TB_SYM_R2_MAXT=4 -DPS_TB_WGS_NW=8 -DPS_TB_RB=8 -DPS_TB_NS=3"
  "c3sym4b|C3:4|f64|$C3T4 -DPS_TB_SYM=2 -DPS_TB_SYM_R2_MAXT=4 -DPS_TB_WGS_NW=8 -DPS_TB_RB=4 -DPS_TB_NS=3"
  "c3old3|C3:3|f64|$C3T3"
  "c2old4|C2:4|f64|$C2T4"
  "c2sleep0|C2:4|f64|$C2T4 -DPS_TB_PROD_SLEEP=0"
  "c2sym4|C2:4|f64|$C2T4 -DPS_TB_SYM=2 -DPS_TB_SYM_WGS=2"
  "c2sym5|C2:5|f64|$C2T5 -DPS_TB_SYM=2 -DPS_TB_SYM_WGS=2"
  "c2old4w8|C2:4|f64|$C2T4 -DPS_TB_WGS=1 -DPS_TB_WGS_NW=8"
  "c5base|C5:4|f32n|$C5T4"
  "c5w8wide|C5:4|f32n|$C5T4 -DPS_TB_WGS_NW=8 -DPS_TB_NARROW=0"
  "c5w8narrow|C5:4|f32n|$C5T4 -DPS_TB_WGS_NW=8"
  "c5w8wide8|C5:4|f32n|$C5T4 -DPS_TB_WGS_NW=8 -DPS_TB_NARROW=0 -DPS_TB_RB=8"
)
if [ "${MODE:-build}" = build ]; then
  for spec in "${VARIANTS[@]}"; do
    IFS='|' read -r v ct unit flags <<< "$spec"
    [ -n "$ONLY" ] && [[ ! " $ONLY " =~ " $v " ]] && continue
    u="ps_kern_${unit}_t${ct##*:}"
    (mkdir -p build/tune/$v &&
     $NV $flags -Xptxas -v -c -o build/tune/$v/$u.o $CSRC/$u.cu > build/tune/$v/ptxas.log 2>&1 &&
     $NV -shared -o build/tune/$v/libps.so $(ls build/obj/*.o | grep -v "/$u.o") build/tune/$v/$u.o &&
     rm -f build/tune/$v/$u.o && echo "$v: $(grep -A2 k_two_step_tb build/tune/$v/ptxas.log | grep -E 'spill|Used' | tr '\n' ' ')") &
  done
  wait
else
  mkdir -p gpurun_out
  for rep in ${REPS:-1 2}; do
    for spec in "${VARIANTS[@]}"; do
      IFS='|' read -r v ct unit flags <<< "$spec"
      [ -n "$ONLY" ] && [[ ! " $ONLY " =~ " $v " ]] && continue
      c=${ct%%:*}; t=${ct##*:}
      PS_LIBRARY="build/tune/$v/libps.so" timeout 200 python bench.py --config $c --steps ${STEPS:-40} \
        --no-e2e --no-cpu --tsteps $t --reps 1 > "gpurun_out/tune_${v}_$rep.json" 2> "gpurun_out/tune_${v}_$rep.err" || true
      python - "$v" "gpurun_out/tune_${v}_$rep.json" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["value"], 1), "GLUP/s", d["clocks"]["sm_mhz"], "MHz")
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
    done
  done
fi
