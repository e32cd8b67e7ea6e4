// ps_tblock.cuh — temporal blocking: TS two-step updates fused in one streaming pass
// (BASELINE config 5, T in {2, 3, 4}).  Included by ps_device.cu.
//
// One pass reads u^k and u^{k-1} once and writes only the last two levels u^{k+TS-1}
// and u^{k+TS}: HBM traffic falls from 3 words per update to 4/TS (+ halos).
//
// Same producer/consumer skeleton as k_two_step_stream (TMA bulk row copies into an
// mbarrier ring, dynamic tiles).  The difference is in the consumers:
//   * each WARP is an independent column unit of 32 lanes x V values (32*V columns) whose
//     outputs are valid on the centre WO = 32V - 2HT columns (HT = R*(TS-1) rounded up
//     to a vector); neighbouring warps overlap by 2HT columns, so no cross-warp exchange
//     is ever needed — the halo is recomputed instead of communicated;
//   * stage t (1..TS) keeps a (2R+1)-row register window of level k+t-1 and produces
//     level k+t R rows behind stage t-1; the -u^{k+t-2} term is the oldest row of the
//     window two stages down (stage 1 takes u^{k-1} from shared memory);
//   * horizontal neighbours of stage outputs come from the adjacent lanes by shuffle;
//   * every stage re-pins the Dirichlet ring (and zeroes rows/cols outside the grid),
//     so each intermediate level is exactly what TS separate launches would produce —
//     results are bitwise equal to the unblocked march.
// Periodic grids: the ghost rows/cols of both inputs must hold wrap-around images to
// depth R*TS (ps_fill_ghosts, or a previous blocked pass, which refreshes them).
#pragma once
// (included inside namespace ps, after the streaming kernel's helpers)

struct TBParams {
  const void* uk;
  const void* ukm1;
  void* out_prev;  // u^{k+TS-1}
  void* out_last;  // u^{k+TS}
  int64_t pitch;
  int32_t rows, cols, ring, row0, grows;
  int32_t rlo, rhi;        // rows this launch finalises
  int32_t gmin, gmax;      // loadable row range [gmin, gmax) (allocation incl. ghosts)
  int32_t cmax;            // loadable columns: element index < cmax (from logical col 0)
  int32_t nstrips, rc, ntiles;
  int32_t reverse;         // walk tiles bottom-up (alternate launches: L2 reuse)
  int32_t row_images;      // periodic: 1 = single slab, also write wrapped row images;
                           // 0 = row slab of a ring (row halos come from the neighbours)
  // row slabs with in-kernel halo delivery (logical-origin pointers of the neighbours'
  // out_prev / out_last levels, null = none): out_last rows [0, R*TS) also land in the
  // slab above at rows up_rows + r, rows [rows - R*TS, rows) in the slab below at r - rows;
  // out_prev likewise with depth R*(TS-1)
  void* hu_prev;
  void* hu_last;
  void* hd_prev;
  void* hd_last;
  int32_t up_rows;
  double c[PS_MAX_TAPS];
  float cf[PS_MAX_TAPS];
};

// VM: 16-byte vectors owned per lane (1 or 2).  Two vectors per lane halve the share of
// recomputed halo columns (f64 T=4: 64/56 -> 128/120) and give each stage twice the
// independent add chains per warp, at twice the window registers.
template <typename T, int NW, int RB, int NS, int R, int TS, int VM = 1>
struct TBGeom {
  static constexpr int VV = Vec<T>::V;                     // elements per 16-byte vector
  static constexpr int V = VM * VV;                        // elements owned per lane
  // Column halo per side.  Stage 1 reads true neighbours from shared memory; each later
  // stage loses R valid columns at each warp edge, so R*(TS-1) (rounded to a lane).
  static constexpr int HT = ((R * (TS - 1) + V - 1) / V) * V;
  static constexpr int WO = 32 * V - 2 * HT;              // valid output columns per warp
  static constexpr int W = NW * WO;                        // output columns per block strip
  static constexpr int LU = W + 2 * HT + 2 * VV;           // u^k row slot (extra vec each side)
  static constexpr int LK = W + 2 * HT;                    // u^{k-1} row slot
  static constexpr size_t smem_bytes =
      size_t(NS) * RB * (LU + LK) * sizeof(T) + 2 * NS * sizeof(uint64_t) + 2 * NS * sizeof(int);
  static_assert(WO > 0, "halo too wide for one warp");
};

template <typename T>
__device__ __forceinline__ T shfl_up1(T x) {
  return __shfl_up_sync(0xffffffffu, x, 1);
}
template <typename T>
__device__ __forceinline__ T shfl_down1(T x) {
  return __shfl_down_sync(0xffffffffu, x, 1);
}

#ifndef PS_TB_PROD_SLEEP
#define PS_TB_PROD_SLEEP 100  // ns the producer sleeps between polls of a ring slot's release
#endif
#ifndef PS_TB_SYM_EDGE
#define PS_TB_SYM_EDGE 1  // shared-product kernels: unrolled body for full ring-adjacent slots
                          // (1: plain passes up to depth 5; 2: every instance)
#endif
#ifndef PS_TB_SYM_HEAD
#define PS_TB_SYM_HEAD 0  // unrolled body for a tile's head slots: 1 = C3 kernel only, 2 = all
                          // (off: C3 f64 T=3 451 -> 458 GLUP/s, C4 within noise, but ptxas
                          // needs 7 more minutes for the second 8-row radius-2 body)
#endif
#ifndef PS_TB_MINB
#define PS_TB_MINB 0  // tuning override: minimum resident blocks per SM (caps registers)
#endif
// Measured (tools/tb_variants.sh): one block of 11 consumer warps + the
// producer per SM beats 3 blocks of 4 + 1 everywhere (C4 468 -> 514, C5 902 -> 1008,
// C3 f64 T=2 321 -> 366 GLUP/s): 12 warps leave 168 registers per thread (3 warps share a
// sub-partition's 16K registers), so the windows fit without spills, and one block keeps
// the whole strip's halo columns in one shared-memory ring.
template <typename T, class S, int TS, bool PER>
constexpr int tb_minb() {
  return PS_TB_MINB > 0 ? PS_TB_MINB : 1;
}

// Narrow windows: stages t >= 1 keep only each lane's own V values per row and fetch the
// neighbours' R columns by shuffle when a row is used (more shuffles, ~(TS-1)(2R+1)·2R
// fewer live registers).  Window 0 stays wide (its neighbours come from shared memory).
#ifndef PS_TB_NARROW
#define PS_TB_NARROW -1
#endif
// Measured: f32 at depth 4 gains (C5 762 -> 834 GLUP/s: 224 -> 168 registers); f64 and
// depth 2 lose to the extra shuffles.
template <typename T, class S, int TS>
__host__ __device__ constexpr bool tb_narrow() {
  return PS_TB_NARROW >= 0 ? PS_TB_NARROW != 0 : (sizeof(T) == 4 && TS == 4);
}

// VM 16-byte vector stores of res[0 .. VM*16/sizeof(T)) to dst, predicated on `pred`
// (an @P STG, not a branch).  Interior tiles only: dst is in bounds and 16-B aligned.
template <typename T, int VM>
__device__ __forceinline__ void st_pred(T* dst, const T* res, bool pred) {
#pragma unroll
  for (int m = 0; m < VM; ++m) {
    if constexpr (sizeof(T) == 8) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %0, 0;\n\t"
          "@p st.global.v2.f64 [%1], {%2, %3};\n\t}" ::"r"(int(pred)),
          "l"(dst + 2 * m), "d"(double(res[2 * m])), "d"(double(res[2 * m + 1])));
    } else {
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %0, 0;\n\t"
          "@p st.global.v4.f32 [%1], {%2, %3, %4, %5};\n\t}" ::"r"(int(pred)),
          "l"(dst + 4 * m), "f"(float(res[4 * m])), "f"(float(res[4 * m + 1])),
          "f"(float(res[4 * m + 2])), "f"(float(res[4 * m + 3])));
    }
  }
}

// Parity of the window column (R + q2) most taps start on: those taps run as packed pairs.
template <class S>
__host__ __device__ constexpr int pair_parity() {
  int n[2] = {0, 0};
  for (int s = 0; s < S::N; ++s) ++n[(S::R + S::q(s, 1)) & 1];
  return n[1] > n[0] ? 1 : 0;
}
#ifndef PS_TB_PAIR
#define PS_TB_PAIR 1  // native f32: FFMA2 for the taps on the majority column parity (0: off)
#endif

// Largest |q2| among the taps of row offset d (how many neighbour columns it reads).
template <class S>
__host__ __device__ constexpr int row_need(int d) {
  int need = 0;
  for (int s = 0; s < S::N; ++s)
    if (S::q(s, 0) == d) need = need > (S::q(s, 1) < 0 ? -S::q(s, 1) : S::q(s, 1))
                                    ? need
                                    : (S::q(s, 1) < 0 ? -S::q(s, 1) : S::q(s, 1));
  return need;
}


// ---------------------------------------------------------------------------
// Shared products (SYM).  The reference's sum adds fl(c_s * u[p + q_s]) tap by tap; the
// product depends only on the input element and the coefficient VALUE, and the named
// schemes give every tap of a symmetry class (centre / axis / corner / distance-2 arm)
// the same coefficient.  So fl(c_axis * u[x]) is one value whether x is read as the
// (-1,0) tap of one output point or the (0,+1) tap of another: the fused kernel computes
// it once per input element and class (P9: 3 multiplies per update instead of 9, P13: 4
// instead of 13) and feeds the same bits into every sum — the additions and their order
// are untouched, so results stay bit-identical to the reference's sequence.
//   * a stage keeps, per non-centre class, the product rows of its last 2R input rows
//     (+R neighbour columns each side, fetched from the adjacent lanes by shuffle — the
//     products travel, not the raw values), the raw own values of those rows (the
//     -u^{k-1} term two stages down) and R partial sums;
//   * an output row's sum is built in table order across R+1 row arrivals: tap s is added
//     when input row (output row + phase(s)) arrives, phase(s) = the largest q1 seen up to
//     tap s (clamped at 0) — exactly the taps whose rows are already in the stage.
// The host checks that the table's coefficients are equal within each class
// (tb_classes_equal); other tables fall back to the unblocked kernels.
constexpr int kTapClasses = 4;  // 0 centre, 1 axis (distance 1), 2 corner, 3 distance-2 arm
template <class S>
__host__ __device__ constexpr int tap_class(int s) {
  const int a = S::q(s, 0) < 0 ? -S::q(s, 0) : S::q(s, 0);
  const int b = S::q(s, 1) < 0 ? -S::q(s, 1) : S::q(s, 1);
  return (a == 0 && b == 0) ? 0 : (a + b == 1) ? 1 : (a == 1 && b == 1) ? 2
         : (a + b == 2) ? 3 : -1;
}
template <class S>
__host__ __device__ constexpr int tap_phase(int s) {
  int ph = 0;
  for (int i = 0; i <= s; ++i) ph = S::q(i, 0) > ph ? S::q(i, 0) : ph;
  return ph;
}
template <class S>
__host__ __device__ constexpr int class_rep(int k) {  // first tap of class k (-1: none)
  for (int s = 0; s < S::N; ++s)
    if (tap_class<S>(s) == k) return s;
  return -1;
}
template <class S>
__host__ __device__ constexpr int class_need(int k) {  // neighbour columns class k reads
  int need = 0;
  for (int s = 0; s < S::N; ++s)
    if (tap_class<S>(s) == k) {
      const int b = S::q(s, 1) < 0 ? -S::q(s, 1) : S::q(s, 1);
      need = b > need ? b : need;
    }
  return need;
}
template <class S>
__host__ __device__ constexpr bool sym_shape() {  // centre first, every tap classified
  if (S::q(0, 0) != 0 || S::q(0, 1) != 0) return false;
  for (int s = 0; s < S::N; ++s)
    if (tap_class<S>(s) < 0 || (s > 0 && tap_class<S>(s) == 0)) return false;
  return true;
}
template <class S>
static bool tb_classes_equal(const ps_table* t) {
  for (int s = 0; s < S::N; ++s) {
    const int rep = class_rep<S>(tap_class<S>(s));
    if (std::memcmp(&t->c[s], &t->c[rep], sizeof(double)) != 0) return false;
  }
  return true;
}
#ifndef PS_TB_SYM
#define PS_TB_SYM 1
#endif
// Where the shared-product path is used (measured on B200, tools/tb_tune.sh):
// every f64 Dirichlet pass whose state fits 8 warpgroup-specialised consumer warps x 232
// registers without spilling: radius 1 at any depth up to 6, radius 2 up to depth 3.
//   C4 (P9, T=4, 200-240 steps under the power cap): 600-605 vs 557 GLUP/s for one product
//   per tap (FP64 instructions per update 19 -> 13); depth 5 — 15 doubles of state per
//   stage is what lets five stages fit — 638; C3 (P13, T=3): 423 vs 382.
// Not used where it measured no better: periodic grids (C2 259 vs 260), the f32 reference
// contract (C5 286 vs 287), radius 2 at depth 4 (1.2 KB of spills: 97-231 vs 360).
// PS_TB_SYM=2 forces it everywhere it can compile, PS_TB_SYM=0 removes it.
#ifndef PS_TB_SYM_R2_MAXT
#define PS_TB_SYM_R2_MAXT 3  // radius 2: deepest fusion whose shared-product state fits
#endif
template <typename T, int A, class S, int TS, bool PER>
__host__ __device__ constexpr bool tb_sym() {
  if (PS_TB_SYM == 0 || !Arith<T, A>::kSplit || !sym_shape<S>()) return false;
  if (S::R > 1 && TS > PS_TB_SYM_R2_MAXT) return false;
  if (PS_TB_SYM == 2) return true;
  return sizeof(T) == 8 && !PER;
}

// HALO: Dirichlet row slab whose boundary rows also go to the neighbours (a separate
// instance, so the plain pass keeps its store path free of the extra checks: they cost
// C5 26 % when compiled into every instance)
// WGS (warpgroup specialisation): warpgroup 0 hands its registers to the others
// (setmaxnreg) and its warp 0 is the producer; the NW consumer warps (NW = 8 or 12) fill
// whole warpgroups, so every SM sub-partition runs the same number of consumers (with a
// single producer warp, 7 or 11 consumers leave one sub-partition a consumer short).
template <int NW>
struct WgsRegs {
  static constexpr int producer = NW == 8 ? 40 : 32;
  static constexpr int consumer = (65536 - 128 * producer) / (NW * 32) / 8 * 8;
};
template <typename T, int A, class S, int TS, bool PER, bool HALO, int NW, int RB, int NS, int VM,
          bool WGS>
__global__ void __launch_bounds__((NW + (WGS ? 4 : 1)) * 32, (tb_minb<T, S, TS, PER>()))
    k_two_step_tb(const __grid_constant__ TBParams p, const int slot) {
  static_assert(!WGS || NW % 4 == 0, "warpgroup specialisation: whole consumer warpgroups");
  constexpr bool NARROW = tb_narrow<T, S, TS>();
  constexpr int R = S::R;
  using G = TBGeom<T, NW, RB, NS, R, TS, VM>;
  constexpr int V = G::V, VV = G::VV, HT = G::HT, WO = G::WO, W = G::W, LU = G::LU, LK = G::LK;
  constexpr int WC = V + 2 * R;  // window row: R left | V own | R right
  static_assert(R <= VV, "neighbour vector must cover the radius");
  using Ar = Arith<T, A>;
  using acc_t = typename Ar::acc_t;
  using coef_t = typename Ar::coef_t;
  using vec_t = typename Vec<T>::type;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* s_uk = reinterpret_cast<T*>(smem_raw);
  T* s_km = s_uk + NS * RB * LU;
  uint64_t* full = reinterpret_cast<uint64_t*>(s_km + NS * RB * LK);
  uint64_t* empty = full + NS;
  int* s_tile = reinterpret_cast<int*>(empty + NS);
  int* s_mlo = s_tile + NS;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    mbar_fence_init();
  }
  __syncthreads();
  pdl_wait();
  pdl_launch_dependents();

  const T* __restrict__ uk = static_cast<const T*>(p.uk);
  const T* __restrict__ ukm1 = static_cast<const T*>(p.ukm1);
  T* __restrict__ out_prev = static_cast<T*>(p.out_prev);
  T* __restrict__ out_last = static_cast<T*>(p.out_last);
  const int64_t pitch = p.pitch;
  constexpr int NE_EXTRA = 2 * R * TS;  // u^k rows beyond the chunk (both sides)

  // ---------------- producer (one thread) ------------------------------------
  // Issues pipeline slot P.g: the TMA row copies of rows [P.mlo, P.mlo + RB) of tile P.tile
  // (or the end sentinel once the tiles are exhausted).  The caller has waited until every
  // consumer warp released that ring stage.  Runs on the producer warp's lane 0.
  struct Prod {
    uint32_t g;
    int tile, mlo;
    bool done;
  };
  auto prod_issue = [&](Prod& P) {
    const uint32_t s = P.g % NS;
    if (P.tile >= p.ntiles) {
      s_tile[s] = -1;
      mbar_arrive(&full[s]);
      P.done = true;
      __threadfence();
      if (atomicAdd(&g_tile_done[slot], 1u) == gridDim.x - 1) {
        g_tile_next[slot] = 0;
        g_tile_done[slot] = 0;
      }
      return;
    }
    // reversed launches walk the tiles bottom-up, so the rows the previous launch wrote
    // last (still in L2) are read first
    const int tid = p.reverse ? p.ntiles - 1 - P.tile : P.tile;
    const int chunk = tid / p.nstrips;
    const int strip = tid - chunk * p.nstrips;
    const int i0 = p.rlo + chunk * p.rc;
    const int i1 = min(i0 + p.rc, p.rhi);
    const int j0 = strip * W;
    // columns: u^k from j0-HT-VV, u^{k-1} from j0-HT; clamp to the allocation row
    const int cu0 = j0 - HT - VV, ck0 = j0 - HT;
    const int nu = max(0, min(LU, p.cmax - cu0)) / VV * VV;
    const int nk = max(0, min(LK, p.cmax - ck0)) / VV * VV;
    const uint32_t ub = uint32_t(nu) * sizeof(T), kb = uint32_t(nk) * sizeof(T);
    const int ne = (i1 - i0) + NE_EXTRA;
    const int mlo = P.mlo;
    s_tile[s] = tid;
    s_mlo[s] = mlo;
    const int mhi = min(mlo + RB, ne);
    uint32_t bytes = 0;
    for (int m = mlo; m < mhi; ++m) {
      const int e = i0 - R * TS + m;
      if (e >= p.gmin && e < p.gmax) bytes += ub;
      const int ek = e - R;
      if (m >= 2 * R && ek >= p.gmin && ek < p.gmax) bytes += kb;
    }
    mbar_arrive_expect_tx(&full[s], bytes);
    const uint64_t pol_uk = l2_policy_evict_normal();
    const uint64_t pol_km = l2_policy_evict_first();
    for (int m = mlo; m < mhi; ++m) {
      const int e = i0 - R * TS + m;
      if (e >= p.gmin && e < p.gmax && ub)
        tma_load_1d(s_uk + (s * RB + (m - mlo)) * LU, uk + int64_t(e) * pitch + cu0, ub,
                    &full[s], pol_uk);
      const int ek = e - R;
      if (m >= 2 * R && ek >= p.gmin && ek < p.gmax && kb)
        tma_load_1d(s_km + (s * RB + (m - mlo)) * LK, ukm1 + int64_t(ek) * pitch + ck0, kb,
                    &full[s], pol_km);
    }
    ++P.g;
    P.mlo += RB;
    if (P.mlo >= ne) {
      P.mlo = 0;
      P.tile = int(gridDim.x + atomicAdd(&g_tile_next[slot], 1u));
    }
  };
  Prod P{0u, int(blockIdx.x), 0, false};

  if (WGS ? (warp < 4) : (warp == NW)) {
    if constexpr (WGS)
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(WgsRegs<NW>::producer) : "memory");
    if ((!WGS || warp == 0) && lane == 0) {
      while (!P.done) {
        const uint32_t k = P.g / NS;
        if (k > 0) mbar_wait_backoff(&empty[P.g % NS], (k - 1) & 1, PS_TB_PROD_SLEEP);
        prod_issue(P);
      }
    }
    return;
  }

  // ---------------- consumers ------------------------------------------------
  if constexpr (WGS)
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(WgsRegs<NW>::consumer) : "memory");
  const int cw = WGS ? warp - 4 : warp;  // consumer warp index
  coef_t c[S::N];
#pragma unroll
  for (int s = 0; s < S::N; ++s) {
    if constexpr (sizeof(coef_t) == sizeof(double))
      c[s] = p.c[s];
    else
      c[s] = p.cf[s];
  }
  // win[t] holds level k+t rows (oldest first), t = 0..TS-1
  T win[TS][2 * R + 1][WC];
#pragma unroll
  for (int t = 0; t < TS; ++t)
#pragma unroll
    for (int r = 0; r < 2 * R + 1; ++r)
#pragma unroll
      for (int x = 0; x < WC; ++x) win[t][r][x] = T(0);

  const int xo = VV + cw * WO + lane * V;  // own values' first column in the u^k slot
  const int xk = cw * WO + lane * V;       // own values' first column in the u^{k-1} slot
  const bool lane_out = (lane * V >= HT) && (lane * V + V <= HT + WO);

  const int gc_lane = cw * WO + lane * V - HT;  // own column relative to the strip start

  auto stage_out = [&](auto interior_tag, int t, const T* minus, int row, int gc0,
                       bool cols_inner, T* res) {
    constexpr bool INTERIOR = decltype(interior_tag)::value;
    // level k+t+1 at `row` from window t; minus = level k+t-1 at the same row
    if (NARROW && t > 0) {  // NOLINT
      // rebuild the neighbour columns of the narrow window by shuffle (only as many as
      // each row offset's taps read)
#pragma unroll
      for (int r = 0; r < 2 * R + 1; ++r) {
#pragma unroll
        for (int q = 0; q < R; ++q) {
          if (q < R - row_need<S>(r - R)) continue;   // column never read
          win[t][r][q] = shfl_up1(win[t][r][R + V - R + q]);
        }
#pragma unroll
        for (int q = 0; q < R; ++q) {
          if (q >= row_need<S>(r - R)) continue;
          win[t][r][R + V + q] = shfl_down1(win[t][r][R + q]);
        }
      }
    }
    acc_t acc[V];
    if constexpr (Ar::kPair && PS_TB_PAIR != 0 && V % 2 == 0) {
      // packed taps: window columns (x, x+1) with x of the parity most taps start on are
      // register pairs, and every tap starting on that parity updates two outputs with one
      // FFMA2; the other taps stay scalar.  Each output still sees its taps in table order.
      constexpr int par = pair_parity<S>();
#pragma unroll
      for (int v = 0; v < V; ++v) acc[v] = Ar::zero();
#pragma unroll
      for (int s = 0; s < S::N; ++s) {
        const int x0 = R + S::q(s, 1);
        if ((x0 & 1) == par) {
#pragma unroll
          for (int v = 0; v < V; v += 2)
            Ar::tap2(acc[v], acc[v + 1], c[s], win[t][R + S::q(s, 0)][x0 + v],
                     win[t][R + S::q(s, 0)][x0 + v + 1]);
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v)
            acc[v] = Ar::tap(acc[v], c[s], win[t][R + S::q(s, 0)][x0 + v]);
        }
      }
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        acc_t a = Ar::zero();
#pragma unroll
        for (int s = 0; s < S::N; ++s)
          a = Ar::tap(a, c[s], win[t][R + S::q(s, 0)][R + v + S::q(s, 1)]);
        acc[v] = a;
      }
    }
    if constexpr (PER || INTERIOR) {
      // periodic (ghosts hold valid images) or a slot whose rows and strip are all off
      // the Dirichlet ring: nothing to mask
      // (packed when the own columns start a register pair of the window)
      if constexpr (Ar::kPair && PS_TB_PAIR != 0 && V % 2 == 0 && (R & 1) == pair_parity<S>()) {
#pragma unroll
        for (int v = 0; v < V; v += 2)
          Ar::two2(res[v], res[v + 1], acc[v], acc[v + 1], minus[v], minus[v + 1]);
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v) res[v] = Ar::two(acc[v], minus[v]);
      }
      return;
    }
    const int gi = p.row0 + row;
    const bool row_in = (gi >= p.ring) && (gi < p.grows - p.ring);
    if (row_in && cols_inner) {
#pragma unroll
      for (int v = 0; v < V; ++v) res[v] = Ar::two(acc[v], minus[v]);
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int gc = gc0 + v;
        const bool in = row_in && (gc >= p.ring) && (gc < p.cols - p.ring);
        res[v] = in ? Ar::two(acc[v], minus[v]) : T(0);
      }
    }
  };

  auto admit = [&](int t, const T* own) {
    // slide window t and admit a new row whose own vector is `own`; neighbours by shuffle
    // (narrow windows slide only the own columns: their neighbour slots are scratch)
#pragma unroll
    for (int r = 0; r < 2 * R; ++r)
#pragma unroll
      for (int x = (NARROW ? R : 0); x < (NARROW ? R + V : WC); ++x) win[t][r][x] = win[t][r + 1][x];
#pragma unroll
    for (int v = 0; v < V; ++v) win[t][2 * R][R + v] = own[v];
    if constexpr (!NARROW) {  // (narrow windows fetch neighbours when a row is used)
#pragma unroll
      for (int q = 0; q < R; ++q) {
        win[t][2 * R][q] = shfl_up1(own[V - R + q]);   // left neighbour's last R values
        win[t][2 * R][R + V + q] = shfl_down1(own[q]);  // right neighbour's first R values
      }
    }
  };

  auto admit_uk = [&](const T* su_row) {
#pragma unroll
    for (int r = 0; r < 2 * R; ++r)
#pragma unroll
      for (int x = 0; x < WC; ++x) win[0][r][x] = win[0][r + 1][x];
    T l[VV], o[V], rr[VV];
    Vec<T>::unpack(*reinterpret_cast<const vec_t*>(su_row + xo - VV), l);
#pragma unroll
    for (int m = 0; m < VM; ++m)
      Vec<T>::unpack(*reinterpret_cast<const vec_t*>(su_row + xo + m * VV), o + m * VV);
    Vec<T>::unpack(*reinterpret_cast<const vec_t*>(su_row + xo + V), rr);
#pragma unroll
    for (int q = 0; q < R; ++q) {
      win[0][2 * R][q] = l[VV - R + q];
      win[0][2 * R][R + V + q] = rr[q];
    }
#pragma unroll
    for (int v = 0; v < V; ++v) win[0][2 * R][R + v] = o[v];
  };

  auto put = [&](T* dst, int gc0, const T* res) {
    if (gc0 + V <= p.cols) {
#pragma unroll
      for (int m = 0; m < VM; ++m)
        reinterpret_cast<vec_t*>(dst)[m] = Vec<T>::pack(res + m * VV);
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v)
        if (gc0 + v < p.cols) dst[v] = res[v];
    }
  };
  // last = true: out_last (halo depth R*TS), else out_prev (depth R*(TS-1))
  auto store_vec = [&](T* base, int row, int gc0, const T* res, bool last) {
    put(base + int64_t(row) * pitch + gc0, gc0, res);
    if constexpr (HALO && !PER) {
      // fused halo delivery: boundary rows also go straight into the neighbours' ghost
      // rows (peer memory over NVLink, ps_two_step_tb_halo)
      void* hu = last ? p.hu_last : p.hu_prev;
      void* hd = last ? p.hd_last : p.hd_prev;
      const int depth = last ? R * TS : R * (TS - 1);
      if (hu && row < depth)
        put(static_cast<T*>(hu) + int64_t(p.up_rows + row) * pitch + gc0, gc0, res);
      if (hd && row >= p.rows - depth)
        put(static_cast<T*>(hd) + int64_t(row - p.rows) * pitch + gc0, gc0, res);
    }
    if constexpr (PER) {
      // refresh wrap-around images to depth D = R*TS (what the next pass loads).  Two
      // copies with constant trip counts, selected once by row_images: a run-time loop
      // bound here kept the image loop rolled and cost the periodic pass 25 % (C2 347 ->
      // 262 GLUP/s between two round-2 commits).
      const int D = R * TS;
      const bool ecol = (gc0 < D) || (gc0 + V > p.cols - D);
      auto images = [&](auto rows_tag) {
        constexpr int RI = decltype(rows_tag)::value ? 1 : 0;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int j = gc0 + v;
          if (j >= p.cols) continue;
#pragma unroll
          for (int a = -RI; a <= RI; ++a)
#pragma unroll
            for (int b = -1; b <= 1; ++b) {
              if (a == 0 && b == 0) continue;
              const int ii = row + a * p.rows;
              const int jj = j + b * p.cols;
              if (ii < -D || ii >= p.rows + D || jj < -D || jj >= p.cols + D) continue;
              base[int64_t(ii) * pitch + jj] = res[v];
            }
        }
      };
      if (p.row_images) {
        if ((row < D) || (row >= p.rows - D) || ecol) images(std::true_type{});
      } else if (ecol) {
        images(std::false_type{});
      }
    }
  };


  if constexpr (tb_sym<T, A, S, TS, PER>()) {
    // ---------------- consumers, shared products (see the note above tap_class) --------
    static_assert(VM == 1 || R == 1, "shared-product state is sized for one or two vectors");
    coef_t cc[kTapClasses];
#pragma unroll
    for (int k = 0; k < kTapClasses; ++k) cc[k] = class_rep<S>(k) >= 0 ? c[class_rep<S>(k) < 0 ? 0 : class_rep<S>(k)] : coef_t(0);
    acc_t part[TS][R][V];                      // sums in flight: part[t][j] = output row a-j
    T rawq[TS][2 * R][V];                      // raw own values of input rows a-2R .. a-1
    acc_t prod[TS][kTapClasses][2 * R][WC];    // product rows a-2R .. a-1 (class 0 unused)
#pragma unroll
    for (int t = 0; t < TS; ++t) {
#pragma unroll
      for (int j = 0; j < R; ++j)
#pragma unroll
        for (int v = 0; v < V; ++v) part[t][j][v] = Ar::zero();
#pragma unroll
      for (int r = 0; r < 2 * R; ++r) {
#pragma unroll
        for (int v = 0; v < V; ++v) rawq[t][r][v] = T(0);
#pragma unroll
        for (int k = 0; k < kTapClasses; ++k)
#pragma unroll
          for (int x = 0; x < WC; ++x) prod[t][k][r][x] = Ar::zero();
      }
    }

    // Stage t takes input row a of level k+t (`own`; stage 0 also its raw neighbours nl/nr
    // from shared memory), finishes the sum of output row a-R of level k+t+1 into `fin`,
    // and returns in `oldest` its raw row a-2R (the next stage's -u term) before sliding.
    auto stage = [&](auto t_tag, const T* own, const T* nl, const T* nr, acc_t* fin,
                     T* oldest) {
      constexpr int t = decltype(t_tag)::value;
      acc_t np[kTapClasses][WC];
#pragma unroll
      for (int k = 1; k < kTapClasses; ++k) {
        if (class_rep<S>(k) < 0) continue;
#pragma unroll
        for (int v = 0; v < V; ++v) np[k][R + v] = Ar::mul(cc[k], own[v]);
#pragma unroll
        for (int q = 0; q < R; ++q) {
          if (q < R - class_need<S>(k)) continue;             // column never read
          if constexpr (t == 0)
            np[k][q] = Ar::mul(cc[k], nl[q]);
          else
            np[k][q] = shfl_up1(np[k][V + q]);                // left lane's last R products
        }
#pragma unroll
        for (int q = 0; q < R; ++q) {
          if (q >= class_need<S>(k)) continue;
          if constexpr (t == 0)
            np[k][R + V + q] = Ar::mul(cc[k], nr[q]);
          else
            np[k][R + V + q] = shfl_down1(np[k][R + q]);      // right lane's first R products
        }
      }
#pragma unroll
      for (int j = R; j >= 0; --j) {
        acc_t a[V];
#pragma unroll
        for (int v = 0; v < V; ++v) a[v] = (j == 0) ? Ar::zero() : part[t][j == 0 ? 0 : j - 1][v];
#pragma unroll
        for (int s = 0; s < S::N; ++s) {
          if (tap_phase<S>(s) != j) continue;
          const int k = tap_class<S>(s);
          const int rel = S::q(s, 0) - j;                     // input row relative to a (<= 0)
#pragma unroll
          for (int v = 0; v < V; ++v) {
            acc_t pv;
            if (k == 0)
              pv = Ar::mul(cc[0], own[v]);
            else if (rel == 0)
              pv = np[k][R + v + S::q(s, 1)];
            else
              pv = prod[t][k][2 * R + rel][R + v + S::q(s, 1)];
            a[v] = Ar::add(a[v], pv);
          }
        }
#pragma unroll
        for (int v = 0; v < V; ++v) {
          if (j == R)
            fin[v] = a[v];
          else
            part[t][j][v] = a[v];
        }
      }
#pragma unroll
      for (int v = 0; v < V; ++v) oldest[v] = rawq[t][0][v];
#pragma unroll
      for (int r = 0; r + 1 < 2 * R; ++r) {
#pragma unroll
        for (int v = 0; v < V; ++v) rawq[t][r][v] = rawq[t][r + 1][v];
#pragma unroll
        for (int k = 1; k < kTapClasses; ++k)
#pragma unroll
          for (int x = 0; x < WC; ++x) prod[t][k][r][x] = prod[t][k][r + 1][x];
      }
#pragma unroll
      for (int v = 0; v < V; ++v) rawq[t][2 * R - 1][v] = own[v];
#pragma unroll
      for (int k = 1; k < kTapClasses; ++k) {
        if (class_rep<S>(k) < 0) continue;
#pragma unroll
        for (int x = 0; x < WC; ++x) prod[t][k][2 * R - 1][x] = np[k][x];
      }
    };

    // sum -> level value: subtract, then the Dirichlet ring / outside-the-grid mask
    auto finish = [&](auto interior_tag, const acc_t* fin, const T* minus, int row, int gc0,
                      bool cols_inner, T* res) {
      constexpr bool INTERIOR = decltype(interior_tag)::value;
      if constexpr (PER || INTERIOR) {
#pragma unroll
        for (int v = 0; v < V; ++v) res[v] = Ar::two(fin[v], minus[v]);
        return;
      }
      const int gi = p.row0 + row;
      const bool row_in = (gi >= p.ring) && (gi < p.grows - p.ring);
      if (row_in && cols_inner) {
#pragma unroll
        for (int v = 0; v < V; ++v) res[v] = Ar::two(fin[v], minus[v]);
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int gc = gc0 + v;
          const bool in = row_in && (gc >= p.ring) && (gc < p.cols - p.ring);
          res[v] = in ? Ar::two(fin[v], minus[v]) : T(0);
        }
      }
    };

    // head_tag: the STEADY body run while the pipeline is still filling (a tile's first
    // slots): every stage runs on whatever its state holds, rows above the tile are never
    // stored, and a stage's state is all valid rows again 2R calls after its input is
    // (sums restart every row, delay lines are 2R rows deep) -- exactly when the rolled
    // body would have switched the stage on.
    auto sym_row = [&](auto steady_tag, auto interior_tag, auto head_tag, const T* su_row,
                       const T* sk_row, int m, int i0, int i1, int j0, bool cols_inner,
                       bool lane_store) {
      constexpr bool STEADY = decltype(steady_tag)::value;
      constexpr bool HEAD = decltype(head_tag)::value;
      static_assert(!HEAD || STEADY, "head slots run the steady body");
      const int e = i0 - R * TS + m;
      const int gc0 = j0 + gc_lane;
      T own[V], nl[VV], nr[VV], res[V], minus[V], oldest[V];
      Vec<T>::unpack(*reinterpret_cast<const vec_t*>(su_row + xo - VV), nl);
#pragma unroll
      for (int mm = 0; mm < VM; ++mm)
        Vec<T>::unpack(*reinterpret_cast<const vec_t*>(su_row + xo + mm * VV), own + mm * VV);
      Vec<T>::unpack(*reinterpret_cast<const vec_t*>(su_row + xo + V), nr);
      bool live = true;   // stage t's output exists once 2R(t+1) rows have flowed
      auto run = [&](auto t_tag) {
        constexpr int t = decltype(t_tag)::value;
        if (!live) return;
        acc_t fin[V];
        T nxt_minus[V];
        // nl holds columns -VV..-1: the R nearest are nl[VV-R..VV)
        stage(t_tag, own, nl + (VV - R), nr, fin, nxt_minus);
        if (!STEADY && m < 2 * R * (t + 1)) {   // state fed, output not yet valid
          live = false;
          return;
        }
        const int row = e - (t + 1) * R;
        if constexpr (t == 0) {
#pragma unroll
          for (int mm = 0; mm < VM; ++mm)
            Vec<T>::unpack(*reinterpret_cast<const vec_t*>(sk_row + xk + mm * VV), minus + mm * VV);
        }
        finish(interior_tag, fin, minus, row, gc0, cols_inner, res);
        constexpr bool PRED_ST = STEADY && decltype(interior_tag)::value && !HALO;
        if constexpr (t == TS - 1) {
          if constexpr (PRED_ST)
            st_pred<T, VM>(out_last + int64_t(row) * pitch + gc0, res,
                           lane_store && (!HEAD || row >= i0));
          else if (lane_store && (STEADY || (row >= i0 && row < i1)))
            store_vec(out_last, row, gc0, res, true);
        } else {
          if constexpr (t == TS - 2) {
            if constexpr (PRED_ST)
              st_pred<T, VM>(out_prev + int64_t(row) * pitch + gc0, res,
                             lane_store && row >= i0 && row < i1);
            else if (lane_store && row >= i0 && row < i1)
              store_vec(out_prev, row, gc0, res, false);
          }
#pragma unroll
          for (int v = 0; v < V; ++v) {
            own[v] = res[v];             // the next stage's input row
            minus[v] = nxt_minus[v];     // and its -u term (this stage's raw row a-2R)
          }
        }
      };
      run(std::integral_constant<int, 0>{});
      if constexpr (TS > 1) run(std::integral_constant<int, 1>{});
      if constexpr (TS > 2) run(std::integral_constant<int, 2>{});
      if constexpr (TS > 3) run(std::integral_constant<int, 3>{});
      if constexpr (TS > 4) run(std::integral_constant<int, 4>{});
      if constexpr (TS > 5) run(std::integral_constant<int, 5>{});
      static_assert(TS <= 6, "add a stage call per extra depth");
    };

    for (uint32_t g = 0;; ++g) {
      const uint32_t s = g % NS;
      const uint32_t k = g / NS;
      mbar_wait(&full[s], k & 1);
      __syncwarp();
      const int tile = s_tile[s];
      if (tile < 0) break;
      const int mlo = s_mlo[s];
      const int chunk = tile / p.nstrips;
      const int strip = tile - chunk * p.nstrips;
      const int i0 = p.rlo + chunk * p.rc;
      const int i1 = min(i0 + p.rc, p.rhi);
      const int j0 = strip * W;
      const int ne = (i1 - i0) + NE_EXTRA;
      const T* su = s_uk + s * RB * LU;
      const T* sk = s_km + s * RB * LK;
      const bool cols_inner = PER || ((j0 - HT >= p.ring) && (j0 + W + HT <= p.cols - p.ring));
      const bool lane_store = lane_out && (j0 + gc_lane < p.cols);
      const bool steady = mlo >= 2 * R * TS && mlo + RB <= ne;
      const int rmin = i0 - R * TS + mlo - TS * R, rmax = i0 - R * TS + mlo + RB - 1 - R;
      constexpr int D = R * TS;
      const bool interior =
          PER ? ((j0 - HT >= D) && (j0 + W + HT <= p.cols - D) && (rmin >= D) && (rmax < p.rows - D))
              : cols_inner && (p.row0 + rmin >= p.ring) && (p.row0 + rmax < p.grows - p.ring);
      if (steady && interior) {
#pragma unroll
        for (int mm = 0; mm < RB; ++mm)
          sym_row(std::true_type{}, std::true_type{}, std::false_type{}, su + mm * LU,
                  sk + mm * LK, mlo + mm, i0, i1, j0, cols_inner, lane_store);
      } else if ((PS_TB_SYM_HEAD == 2 || (PS_TB_SYM_HEAD == 1 && R == 2 && TS == 3)) && !HALO &&
                 !PER && interior && mlo + RB <= ne) {
        // a full head slot of a tile off the ring: the unrolled body with row-checked stores
        // instead of the rolled one (2 of a tile's slots, ~3x the steady cost each).  Only
        // where it measured a gain worth a second copy of the unrolled body: C3 f64 T=3
        // 451 -> 458 GLUP/s; C4 T=5 within noise (750 vs 728-758) for twice the compile time.
#pragma unroll
        for (int mm = 0; mm < RB; ++mm)
          sym_row(std::true_type{}, std::true_type{}, std::true_type{}, su + mm * LU,
                  sk + mm * LK, mlo + mm, i0, i1, j0, cols_inner, lane_store);
      } else if ((PS_TB_SYM_EDGE == 2 || (PS_TB_SYM_EDGE == 1 && !HALO && TS <= 5)) && steady) {
        // full slots touching the Dirichlet ring (first/last strips and chunks): unrolled
        // too, masks and plain stores kept (C4 +2 %, C3 +8 %).  Radius 2 unrolls one 2R-row
        // rotation of the delay lines at a time: the 8-row body takes ptxas 8 minutes.
        constexpr int EU = (R == 1 || RB % (2 * R) != 0) ? RB : 2 * R;
#pragma unroll 1
        for (int m0 = 0; m0 < RB; m0 += EU) {
#pragma unroll
          for (int mm = 0; mm < EU; ++mm)
            sym_row(std::true_type{}, std::false_type{}, std::false_type{}, su + (m0 + mm) * LU,
                    sk + (m0 + mm) * LK, mlo + m0 + mm, i0, i1, j0, cols_inner, lane_store);
        }
      } else {
        // tile heads/tails and slots touching the ring (or the image bands): one rolled
        // body with every check (a few percent of the slots on the large grids)
#pragma unroll 1
        for (int mm = 0; mm < min(RB, ne - mlo); ++mm)
          sym_row(std::false_type{}, std::false_type{}, std::false_type{}, su + mm * LU,
                  sk + mm * LK, mlo + mm, i0, i1, j0, cols_inner, lane_store);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  } else {
  // ---------------- consumers, one product per tap (NATIVE f32, PS_TB_SYM=0) -----------
  // One u^k row through every stage.  STEADY: all TS windows are full and the final row
  // lies inside the tile (no per-stage checks, so the unrolled window rotation compiles
  // to register renaming).  Otherwise stage t+1 runs only once window t is full.
  auto row_step = [&](auto steady_tag, auto interior_tag, const T* su_row, const T* sk_row,
                      int m, int i0, int i1, int j0, bool cols_inner, bool lane_store) {
    constexpr bool STEADY = decltype(steady_tag)::value;
    admit_uk(su_row);
    const int e = i0 - R * TS + m;
    const int gc0 = j0 + gc_lane;
#pragma unroll
    for (int t = 0; t < TS; ++t) {
      if (!STEADY && m < 2 * R * (t + 1)) break;
      const int row = e - (t + 1) * R;
      T minus[V];
      if (t == 0) {
#pragma unroll
        for (int m = 0; m < VM; ++m)
          Vec<T>::unpack(*reinterpret_cast<const vec_t*>(sk_row + xk + m * VV), minus + m * VV);
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v) minus[v] = win[t - 1][0][R + v];
      }
      T res[V];
      stage_out(interior_tag, t, minus, row, gc0, cols_inner, res);
      // steady interior slots of a plain pass store with predicated vector stores: no
      // branch (and no reconvergence point) splits the unrolled rows, so the scheduler
      // can overlap one stage's dependent add chain with the next row's products
      // (periodic: interior = off the wrap-around image bands, so no image stores either)
      constexpr bool PRED_ST = STEADY && decltype(interior_tag)::value && !HALO;
      if (t == TS - 1) {
        if constexpr (PRED_ST)
          st_pred<T, VM>(out_last + int64_t(row) * pitch + gc0, res, lane_store);
        else if (lane_store && (STEADY || (row >= i0 && row < i1)))
          store_vec(out_last, row, gc0, res, true);
      } else {
        if (t == TS - 2) {
          if constexpr (PRED_ST)
            st_pred<T, VM>(out_prev + int64_t(row) * pitch + gc0, res,
                           lane_store && row >= i0 && row < i1);
          else if (lane_store && row >= i0 && row < i1)
            store_vec(out_prev, row, gc0, res, false);
        }
        admit(t + 1, res);
      }
    }
  };

  for (uint32_t g = 0;; ++g) {
    const uint32_t s = g % NS;
    const uint32_t k = g / NS;
    mbar_wait(&full[s], k & 1);
    __syncwarp();  // converged from here on: the shuffles need no divergence checks
    const int tile = s_tile[s];
    if (tile < 0) break;
    const int mlo = s_mlo[s];
    const int chunk = tile / p.nstrips;
    const int strip = tile - chunk * p.nstrips;
    const int i0 = p.rlo + chunk * p.rc;
    const int i1 = min(i0 + p.rc, p.rhi);
    const int j0 = strip * W;
    const int ne = (i1 - i0) + NE_EXTRA;
    const T* su = s_uk + s * RB * LU;
    const T* sk = s_km + s * RB * LK;
    // whole strip away from the global ring and the right edge: no column masks
    const bool cols_inner = PER || ((j0 - HT >= p.ring) && (j0 + W + HT <= p.cols - p.ring));
    const bool lane_store = lane_out && (j0 + gc_lane < p.cols);
    const bool steady = mlo >= 2 * R * TS && mlo + RB <= ne;
    // every stage output row of this slot lies in [row0+rmin, row0+rmax]
    const int rmin = i0 - R * TS + mlo - TS * R, rmax = i0 - R * TS + mlo + RB - 1 - R;
    constexpr int D = R * TS;  // periodic: depth of the image bands each pass rewrites
    const bool interior =
        PER ? ((j0 - HT >= D) && (j0 + W + HT <= p.cols - D) && (rmin >= D) && (rmax < p.rows - D))
            : cols_inner && (p.row0 + rmin >= p.ring) && (p.row0 + rmax < p.grows - p.ring);
    if (steady && interior) {
#pragma unroll
      for (int mm = 0; mm < RB; ++mm)
        row_step(std::true_type{}, std::true_type{}, su + mm * LU, sk + mm * LK, mlo + mm, i0, i1,
                 j0, cols_inner, lane_store);
    } else if (steady) {
#pragma unroll
      for (int mm = 0; mm < RB; ++mm)
        row_step(std::true_type{}, std::false_type{}, su + mm * LU, sk + mm * LK, mlo + mm, i0,
                 i1, j0, cols_inner, lane_store);
    } else {
#pragma unroll 1
      for (int mm = 0; mm < min(RB, ne - mlo); ++mm)
        row_step(std::false_type{}, std::false_type{}, su + mm * LU, sk + mm * LK, mlo + mm, i0,
                 i1, j0, cols_inner, lane_store);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  }  // (one product per tap)
}
