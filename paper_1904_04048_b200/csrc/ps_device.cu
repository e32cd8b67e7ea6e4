// ps_device.cu — sm_100a kernels and the C-ABI of libps.so (declared in include/ps.h).
//
// Hot path: the two-step update u^{k+1} = A(u^k) - u^{k-1} of the reference's
// simulator.py:147-205, as a persistent, warp-specialised row-streaming kernel:
//   * one producer warp issues TMA bulk copies (cp.async.bulk -> UBLKCP) of u^k row
//     segments (strip + 16-byte halo each side) and u^{k-1} row segments into a ring
//     of NS shared-memory stages guarded by mbarrier transaction counts;
//   * NW consumer warps slide a (2R+1)-row register window down the strip: every u^k
//     element crosses HBM once and shared memory once, vertical taps come from
//     registers, horizontal taps from the 16-byte neighbour vectors held beside it;
//   * results leave as 16-byte vector stores; periodic edge points also write their
//     wrap-around images so the next step streams plain rows.
// Tap order and arithmetic follow the reference bit for bit (ps_arith.cuh).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <utility>
#include <vector>

#include "ps.h"
#include "ps_arith.cuh"
#include "ps_ptx.cuh"

// Streaming-kernel geometry (tuning builds override with -D): consumer warps per
// block, rows per pipeline stage for radius 1 / radius 2, pipeline stages.
#ifndef PS_NW
#define PS_NW 8
#endif
#ifndef PS_RB1
#define PS_RB1 4
#endif
#ifndef PS_RB2
#define PS_RB2 4
#endif
#ifndef PS_NS
#define PS_NS 3
#endif

namespace ps {

static std::atomic<int64_t> g_launches{0};
static std::atomic<uint64_t> g_launch_seq{0};

// ---------------------------------------------------------------------------
// Stencil shapes: compile-time tap lists in the reference's dict order
// (scheme.py:54-83 keeps Lagrange-node order; C9 follows isotropic_nine_point
// insertion order scheme.py:100-124).  Coefficients stay runtime values.
// ---------------------------------------------------------------------------
#define PS_SHAPE(NAME, NT, RAD, ...)                                            \
  struct NAME {                                                                 \
    static constexpr int N = NT;                                                \
    static constexpr int R = RAD;                                               \
    __host__ __device__ static constexpr int q(int s, int axis) {               \
      constexpr int t[2 * NT] = {__VA_ARGS__};                                  \
      return t[2 * s + axis];                                                   \
    }                                                                           \
  };
PS_SHAPE(ShapeP5, 5, 1, 0, 0, -1, 0, 0, -1, 1, 0, 0, 1)
PS_SHAPE(ShapeP9, 9, 1, 0, 0, -1, 0, 0, -1, -1, -1, 1, 0, 0, 1, 1, -1, -1, 1, 1, 1)
PS_SHAPE(ShapeC9, 9, 1, 0, 0, -1, 0, 0, -1, 1, 0, 0, 1, -1, -1, 1, -1, -1, 1, 1, 1)
PS_SHAPE(ShapeP13, 13, 2, 0, 0, -1, 0, 0, -1, -1, -1, 1, 0, 0, 1, 1, -1, -1, 1, -2, 0, 0, -2,
         1, 1, 2, 0, 0, 2)
#undef PS_SHAPE

template <class S>
static bool shape_matches(const ps_table* t) {
  if (t->ntaps != S::N) return false;
  for (int s = 0; s < S::N; ++s)
    if (t->q1[s] != S::q(s, 0) || t->q2[s] != S::q(s, 1)) return false;
  return true;
}

template <typename T>
struct Vec;
template <>
struct Vec<double> {
  using type = double2;
  static constexpr int V = 2;
  __device__ __forceinline__ static void unpack(const type& x, double* d) {
    d[0] = x.x;
    d[1] = x.y;
  }
  __device__ __forceinline__ static type pack(const double* d) { return make_double2(d[0], d[1]); }
};
template <>
struct Vec<float> {
  using type = float4;
  static constexpr int V = 4;
  __device__ __forceinline__ static void unpack(const type& x, float* d) {
    d[0] = x.x;
    d[1] = x.y;
    d[2] = x.z;
    d[3] = x.w;
  }
  __device__ __forceinline__ static type pack(const float* d) {
    return make_float4(d[0], d[1], d[2], d[3]);
  }
};

// ---------------------------------------------------------------------------
// Streaming two-step kernel
// ---------------------------------------------------------------------------
struct StreamParams {
  const void* uk;    // logical (0,0) of u^k
  const void* ukm1;  // logical (0,0) of u^{k-1}
  void* ukp1;        // logical (0,0) of u^{k+1}
  int64_t pitch;
  int32_t rows, cols, ring;
  int32_t row0, grows;     // slab: global index of row 0, global row count
  int32_t rlo, rhi;        // rows this launch updates
  int32_t row_images;      // periodic, single slab: also write wrapped row images
  int32_t nstrips, rc, ntiles;
  // row slabs with in-kernel halo delivery: the first/last R output rows are also
  // stored into the neighbours' ghost rows (peer pointers to their u^{k+1} origins)
  void* halo_up;           // neighbour above: rows [0,R) -> its rows [up_rows, up_rows+R)
  void* halo_dn;           // neighbour below: rows [rows-R,rows) -> its rows [-R, 0)
  int32_t up_rows;
  int32_t reverse;          // walk tiles bottom-up (alternate launches: L2 reuse)
  // periodic images: 1 = read u^{k-1} at each image position (the drop-in's possibly
  // inconsistent alias, simulator.py:184); 0 = images of u^{k-1} are copies of its core
  // (every level the march produces), so the image value equals the core value
  int32_t img_exact;
  double tau;              // VP launches: output -fl(tau * acc) (first step, velocity half)
  float tauf;
  double c[PS_MAX_TAPS];
  float cf[PS_MAX_TAPS];
};

template <typename T, int NW, int RB, int NS>
struct StreamGeom {
  static constexpr int V = Vec<T>::V;
  static constexpr int W = NW * 32 * V;  // columns per strip
  static constexpr int SU = W + 2 * V;   // u^k slot: strip + one 16-byte vector each side
  static constexpr size_t smem_bytes =
      size_t(NS) * RB * (SU + W) * sizeof(T) + 2 * NS * sizeof(uint64_t) + 2 * NS * sizeof(int);
};

// Dynamic tile scheduler: one counter pair per in-flight launch (slot = launch
// sequence number mod kSlots).  The last block to finish resets its slot, so the next
// launch that reuses it (kSlots launches later) starts from zero.
constexpr int kSlots = 1024;
__device__ unsigned int g_tile_next[kSlots];
__device__ unsigned int g_tile_done[kSlots];

// VP = true: the first step's velocity half, -fl(tau * A_v(v0)), written where a second
// (ordinary) launch with the displacement table reads it as "u^{k-1}"; no u^{k-1} loads.
template <typename T, int A, class S, bool PER, int NW, int RB, int NS, bool VP = false>
__global__ void __launch_bounds__((NW + 1) * 32)
    k_two_step_stream(const __grid_constant__ StreamParams p, const int slot) {
  using G = StreamGeom<T, NW, RB, NS>;
  constexpr int V = G::V, W = G::W, SU = G::SU;
  constexpr int R = S::R;
  static_assert(R <= V, "halo vector must cover the stencil radius");
  using Ar = Arith<T, A>;
  using acc_t = typename Ar::acc_t;
  using coef_t = typename Ar::coef_t;
  using vec_t = typename Vec<T>::type;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* s_uk = reinterpret_cast<T*>(smem_raw);
  T* s_km = s_uk + NS * RB * SU;
  uint64_t* full = reinterpret_cast<uint64_t*>(s_km + NS * RB * W);
  uint64_t* empty = full + NS;
  int* s_tile = reinterpret_cast<int*>(empty + NS);  // tile of each stage (-1: stop)
  int* s_mlo = s_tile + NS;                           // first window row of each stage

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
  pdl_wait();                 // predecessor's levels complete and visible
  pdl_launch_dependents();    // successor may start its prologue as our blocks drain

  const T* __restrict__ uk = static_cast<const T*>(p.uk);
  const T* __restrict__ ukm1 = static_cast<const T*>(p.ukm1);
  T* __restrict__ ukp1 = static_cast<T*>(p.ukp1);
  const int64_t pitch = p.pitch;

  if (warp == NW) {
    // ---------------- producer: one elected lane streams rows via TMA ----------
    if (lane == 0) {
      // u^k rows are re-read as halos by the neighbouring tiles: keep them normal in
      // L2; u^{k-1} is read exactly once: evict first.
      const uint64_t pol_uk = l2_policy_evict_normal();
      const uint64_t pol_km = l2_policy_evict_first();
      uint32_t g = 0;
      int tile = blockIdx.x;
      while (tile < p.ntiles) {
        // reversed launches walk the tiles bottom-up, so the rows the previous launch
        // wrote last (still in L2) are read first
        const int tid = p.reverse ? p.ntiles - 1 - tile : tile;
        const int chunk = tid / p.nstrips;
        const int strip = tid - chunk * p.nstrips;
        const int i0 = p.rlo + chunk * p.rc;
        const int i1 = min(i0 + p.rc, p.rhi);
        const int j0 = strip * W;
        const int wv = ((min(W, p.cols - j0) + V - 1) / V) * V;
        const uint32_t ukb = uint32_t(wv + 2 * V) * sizeof(T);
        const uint32_t kmb = uint32_t(wv) * sizeof(T);
        const int ne = (i1 - i0) + 2 * R;
        for (int mlo = 0; mlo < ne; mlo += RB, ++g) {
          const uint32_t s = g % NS;
          const uint32_t k = g / NS;
          if (k > 0) mbar_wait(&empty[s], (k - 1) & 1);
          s_tile[s] = tid;
          s_mlo[s] = mlo;
          const int mhi = min(mlo + RB, ne);
          const int nk = VP ? 0 : max(0, mhi - max(mlo, 2 * R));
          mbar_arrive_expect_tx(&full[s], uint32_t(mhi - mlo) * ukb + uint32_t(nk) * kmb);
          for (int m = mlo; m < mhi; ++m) {
            const int64_t e = int64_t(i0) - R + m;
            tma_load_1d(s_uk + (s * RB + (m - mlo)) * SU, uk + e * pitch + j0 - V, ukb, &full[s],
                        pol_uk);
            if (!VP && m >= 2 * R) {
              const int64_t i = int64_t(i0) + m - 2 * R;
              tma_load_1d(s_km + (s * RB + (m - mlo)) * W, ukm1 + i * pitch + j0, kmb, &full[s],
                          pol_km);
            }
          }
        }
        tile = int(gridDim.x + atomicAdd(&g_tile_next[slot], 1u));
      }
      // sentinel stage: tells the consumers to stop
      const uint32_t s = g % NS;
      const uint32_t k = g / NS;
      if (k > 0) mbar_wait(&empty[s], (k - 1) & 1);
      s_tile[s] = -1;
      mbar_arrive(&full[s]);
      __threadfence();
      if (atomicAdd(&g_tile_done[slot], 1u) == gridDim.x - 1) {
        g_tile_next[slot] = 0;
        g_tile_done[slot] = 0;
      }
    }
    return;
  }

  // ---------------- consumers ------------------------------------------------
  coef_t c[S::N];
#pragma unroll
  for (int s = 0; s < S::N; ++s) {
    if constexpr (sizeof(coef_t) == sizeof(double))
      c[s] = p.c[s];
    else
      c[s] = p.cf[s];
  }
  T w[2 * R + 1][3 * V];  // rows i-R..i+R; cols: left vec | own vec | right vec
#pragma unroll
  for (int r = 0; r < 2 * R + 1; ++r)
#pragma unroll
    for (int x = 0; x < 3 * V; ++x) w[r][x] = T(0);

  const int tcol = threadIdx.x * V;

  auto row_step = [&](const T* su_row, const T* sk_row, int m, int i0, int jv, bool active,
                      bool cols_inner) {
    // slide the window and admit u^k row (i0 - R + m)
#pragma unroll
    for (int r = 0; r < 2 * R; ++r)
#pragma unroll
      for (int x = 0; x < 3 * V; ++x) w[r][x] = w[r + 1][x];
    {
      const vec_t a = *reinterpret_cast<const vec_t*>(su_row + tcol);
      const vec_t b = *reinterpret_cast<const vec_t*>(su_row + tcol + V);
      const vec_t d = *reinterpret_cast<const vec_t*>(su_row + tcol + 2 * V);
      Vec<T>::unpack(a, &w[2 * R][0]);
      Vec<T>::unpack(b, &w[2 * R][V]);
      Vec<T>::unpack(d, &w[2 * R][2 * V]);
    }
    if (m < 2 * R || !active) return;
    const int i = i0 + m - 2 * R;
    T km[V];
    if constexpr (!VP) Vec<T>::unpack(*reinterpret_cast<const vec_t*>(sk_row + tcol), km);
    acc_t acc[V];
    T out[V];
    auto fin = [&](acc_t a, T kmv) -> T {
      if constexpr (VP) {
        if constexpr (sizeof(T) == sizeof(double))
          return Ar::vpart(a, p.tau);
        else
          return Ar::vpart(a, p.tauf);
      } else {
        return Ar::two(a, kmv);
      }
    };
#pragma unroll
    for (int v = 0; v < V; ++v) {
      acc_t a = Ar::zero();
#pragma unroll
      for (int s = 0; s < S::N; ++s) a = Ar::tap(a, c[s], w[R + S::q(s, 0)][V + v + S::q(s, 1)]);
      acc[v] = a;
    }
    T* dst = ukp1 + int64_t(i) * pitch + jv;
    if constexpr (PER) {
#pragma unroll
      for (int v = 0; v < V; ++v) out[v] = fin(acc[v], km[v]);
    } else {
      const int gi = p.row0 + i;
      const bool row_in = (gi >= p.ring) && (gi < p.grows - p.ring);
      if (row_in && cols_inner) {
#pragma unroll
        for (int v = 0; v < V; ++v) out[v] = fin(acc[v], km[v]);
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int j = jv + v;
          const bool in = row_in && (j >= p.ring) && (j < p.cols - p.ring);
          out[v] = in ? fin(acc[v], km[v]) : T(0);
        }
      }
    }
    if (jv + V <= p.cols) {
      *reinterpret_cast<vec_t*>(dst) = Vec<T>::pack(out);
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v)
        if (jv + v < p.cols) dst[v] = out[v];
    }
    if constexpr (!PER) {
      // in-kernel halo delivery over NVLink (peer-mapped pointers; plain stores)
      T* peer = nullptr;
      if (i < R && p.halo_up)
        peer = static_cast<T*>(p.halo_up) + int64_t(p.up_rows + i) * pitch + jv;
      else if (i >= p.rows - R && p.halo_dn)
        peer = static_cast<T*>(p.halo_dn) + int64_t(i - p.rows) * pitch + jv;
      if (peer) {
        if (jv + V <= p.cols) {
          *reinterpret_cast<vec_t*>(peer) = Vec<T>::pack(out);
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v)
            if (jv + v < p.cols) peer[v] = out[v];
        }
      }
    }
    if constexpr (PER) {
      const bool erow = p.row_images && ((i < R) || (i >= p.rows - R));
      const bool ecol = (jv < R) || (jv + V > p.cols - R);
      if (erow || ecol) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int j = jv + v;
          if (j >= p.cols) continue;
          for (int a = -p.row_images; a <= p.row_images; ++a)
            for (int b = -1; b <= 1; ++b) {
              if (a == 0 && b == 0) continue;
              const int ii = i + a * p.rows;
              const int jj = j + b * p.cols;
              if (ii < -R || ii >= p.rows + R || jj < -R || jj >= p.cols + R) continue;
              const int64_t o = int64_t(ii) * pitch + jj;
              ukp1[o] = (!VP && p.img_exact) ? Ar::two(acc[v], ukm1[o]) : out[v];
            }
        }
      }
    }
  };

  for (uint32_t g = 0;; ++g) {
    const uint32_t s = g % NS;
    const uint32_t k = g / NS;
    mbar_wait(&full[s], k & 1);
    const int tile = s_tile[s];
    if (tile < 0) break;
    const int mlo = s_mlo[s];
    const int chunk = tile / p.nstrips;
    const int strip = tile - chunk * p.nstrips;
    const int i0 = p.rlo + chunk * p.rc;
    const int i1 = min(i0 + p.rc, p.rhi);
    const int j0 = strip * W;
    const int jv = j0 + tcol;
    const bool active = jv < p.cols;
    const bool cols_inner = (j0 >= p.ring) && (j0 + W <= p.cols - p.ring);
    const int ne = (i1 - i0) + 2 * R;
    const T* su = s_uk + s * RB * SU;
    const T* sk = s_km + s * RB * W;
    if (mlo + RB <= ne) {
#pragma unroll
      for (int mm = 0; mm < RB; ++mm)
        row_step(su + mm * SU, sk + mm * W, mlo + mm, i0, jv, active, cols_inner);
    } else {
      for (int mm = 0; mm < ne - mlo; ++mm)
        row_step(su + mm * SU, sk + mm * W, mlo + mm, i0, jv, active, cols_inner);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

#include "ps_tblock.cuh"
#include "ps_errsum.cuh"

// ---------------------------------------------------------------------------
// Generic kernels (any tap list within the ghost width; first step; images)
// ---------------------------------------------------------------------------
struct GenTable {
  int32_t ntaps;
  int32_t q1[PS_MAX_TAPS], q2[PS_MAX_TAPS];
  double c[PS_MAX_TAPS];
  float cf[PS_MAX_TAPS];
};

struct GenParams {
  const void* a;  // u^k (two-step) or u0 (first step)
  const void* b;  // u^{k-1} (two-step) or v0 (first step)
  void* out;
  int64_t pitch;
  int32_t rows, cols, ring, radius;
  int32_t row0, grows, rlo, rhi, row_images;
  void* halo_up;
  void* halo_dn;
  int32_t up_rows;
  double tau;
  float tauf;
  GenTable ta, tb;
};

template <typename T, int A>
__device__ __forceinline__ typename Arith<T, A>::acc_t gen_acc(const GenTable& t, const T* u,
                                                               int64_t pitch, int i, int j) {
  using Ar = Arith<T, A>;
  typename Ar::acc_t acc = Ar::zero();
  for (int s = 0; s < t.ntaps; ++s) {
    const T x = u[int64_t(i + t.q1[s]) * pitch + (j + t.q2[s])];
    if constexpr (sizeof(typename Ar::coef_t) == sizeof(double))
      acc = Ar::tap(acc, t.c[s], x);
    else
      acc = Ar::tap(acc, t.cf[s], x);
  }
  return acc;
}

template <typename T, int A, bool PER, bool FIRST>
__global__ void __launch_bounds__(256) k_generic(const __grid_constant__ GenParams p) {
  using Ar = Arith<T, A>;
  const T* __restrict__ ua = static_cast<const T*>(p.a);
  const T* __restrict__ ub = static_cast<const T*>(p.b);
  T* __restrict__ out = static_cast<T*>(p.out);
  const int64_t pitch = p.pitch;
  for (int i = p.rlo + blockIdx.y * blockDim.y + threadIdx.y; i < p.rhi;
       i += gridDim.y * blockDim.y) {
    const int gi = p.row0 + i;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < p.cols;
         j += gridDim.x * blockDim.x) {
      const int64_t o = int64_t(i) * pitch + j;
      const bool in = PER || ((gi >= p.ring) && (gi < p.grows - p.ring) && (j >= p.ring) &&
                              (j < p.cols - p.ring));
      if (!in) {
        out[o] = T(0);
        if constexpr (!PER) {
          if (i < p.radius && p.halo_up)
            static_cast<T*>(p.halo_up)[int64_t(p.up_rows + i) * pitch + j] = T(0);
          else if (i >= p.rows - p.radius && p.halo_dn)
            static_cast<T*>(p.halo_dn)[int64_t(i - p.rows) * pitch + j] = T(0);
        }
        continue;
      }
      const auto acc = gen_acc<T, A>(p.ta, ua, pitch, i, j);
      T val;
      typename Ar::acc_t accb{};
      if constexpr (FIRST) {
        accb = gen_acc<T, A>(p.tb, ub, pitch, i, j);
        if constexpr (sizeof(T) == sizeof(double))
          val = Ar::first(acc, accb, p.tau);
        else
          val = Ar::first(acc, accb, p.tauf);
      } else {
        val = Ar::two(acc, ub[o]);
      }
      out[o] = val;
      if constexpr (!PER) {
        if (i < p.radius && p.halo_up)
          static_cast<T*>(p.halo_up)[int64_t(p.up_rows + i) * pitch + j] = val;
        else if (i >= p.rows - p.radius && p.halo_dn)
          static_cast<T*>(p.halo_dn)[int64_t(i - p.rows) * pitch + j] = val;
      }
      if constexpr (PER) {
        // images within the stencil radius, and always the first one (the reference's
        // alias row/col n), even for a radius-0 table
        const int R = max(p.radius, 1);
        if ((p.row_images && (i < R || i >= p.rows - R)) || j < R || j >= p.cols - R) {
          const int aw = p.row_images ? (R + p.rows - 1) / p.rows : 0;
          const int bw = (R + p.cols - 1) / p.cols;
          for (int a = -aw; a <= aw; ++a)
            for (int b = -bw; b <= bw; ++b) {
              if (a == 0 && b == 0) continue;
              const int ii = i + a * p.rows;
              const int jj = j + b * p.cols;
              if (ii < -R || ii >= p.rows + R || jj < -R || jj >= p.cols + R) continue;
              const int64_t oo = int64_t(ii) * pitch + jj;
              if constexpr (FIRST)
                out[oo] = val;
              else
                out[oo] = Ar::two(acc, ub[oo]);
            }
        }
      }
    }
  }
}

// Periodic image refresh over the padding band (simulator.py:135-138).
template <typename T>
__global__ void __launch_bounds__(256)
    k_fill_ghosts(T* base, int64_t pitch, int32_t rows, int32_t cols, int32_t G, int32_t keep) {
  const int64_t wfull = int64_t(cols) + 2 * G;
  const int64_t n_tb = 2 * int64_t(G) * wfull;  // top + bottom bands
  const int64_t n_lr = 2 * int64_t(G) * rows;   // left + right bands
  const int64_t total = n_tb + n_lr;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total;
       t += int64_t(gridDim.x) * blockDim.x) {
    int64_t ii, jj;
    if (t < n_tb) {
      const int64_t r = t / wfull;
      jj = (t - r * wfull) - G;
      ii = r < G ? r - G : rows + (r - G);
    } else {
      const int64_t u = t - n_tb;
      const int64_t r = u / (2 * G);
      const int64_t x = u - r * 2 * G;
      ii = r;
      jj = x < G ? x - G : cols + (x - G);
    }
    if (keep && ii >= 0 && ii <= rows && jj >= 0 && jj <= cols) continue;
    const int64_t si = ((ii % rows) + rows) % rows;
    const int64_t sj = ((jj % cols) + cols) % cols;
    base[ii * pitch + jj] = base[si * pitch + sj];
  }
}

// Gaussian-sum initial data (BASELINE configs 3-5).
constexpr int kMaxGauss = 512;
struct GaussParams {
  int32_t K;
  int32_t rows, cols, row0;
  int64_t pitch;
  double n;
  double cx[kMaxGauss], cy[kMaxGauss], w2[kMaxGauss], amp[kMaxGauss];
};

template <typename T>
__global__ void __launch_bounds__(256) k_gaussian(const __grid_constant__ GaussParams p, T* base) {
  for (int i = blockIdx.y * blockDim.y + threadIdx.y; i < p.rows; i += gridDim.y * blockDim.y) {
    const double x1 = double(p.row0 + i) / p.n;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < p.cols;
         j += gridDim.x * blockDim.x) {
      const double x2 = double(j) / p.n;
      double acc = 0.0;
      for (int k = 0; k < p.K; ++k) {
        const double d1 = __dsub_rn(x1, p.cx[k]);
        const double d2 = __dsub_rn(x2, p.cy[k]);
        const double r2 = __dadd_rn(__dmul_rn(d1, d1), __dmul_rn(d2, d2));
        acc = __dadd_rn(acc, __dmul_rn(p.amp[k], exp(-__ddiv_rn(r2, p.w2[k]))));
      }
      base[int64_t(i) * p.pitch + j] = T(acc);
    }
  }
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
struct DevInfo {
  int nsm = 0;
};
static DevInfo dev_info() {
  static std::mutex mu;
  static DevInfo cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cache[dev].nsm == 0) cudaDeviceGetAttribute(&cache[dev].nsm, cudaDevAttrMultiProcessorCount, dev);
  return cache[dev];
}

static int env_int(const char* name, int dflt) {
  const char* s = std::getenv(name);
  return (s && *s) ? std::atoi(s) : dflt;
}

static ps_status last_cuda_status() {
  return cudaGetLastError() == cudaSuccess ? PS_OK : PS_ERR_CUDA;
}

// Launch with programmatic stream serialization (PDL) unless PS_PDL=0: the kernel's
// blocks may be scheduled while the previous kernel in the stream drains; the kernel
// itself waits (griddepcontrol.wait) before reading anything the predecessor wrote.
template <typename Params>
static cudaError_t launch_pdl(void (*kern)(Params, int), int grid, int block, size_t smem,
                              cudaStream_t st, const Params& p, int slot) {
  static const bool pdl = env_int("PS_PDL", 1) != 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(unsigned(block));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, p, slot);
}

template <typename T>
static T* at_origin(const ps_grid* g, const void* level) {
  return static_cast<T*>(const_cast<void*>(level)) + g->origin;
}

static int table_radius(const ps_table* t) {
  int r = 0;
  for (int s = 0; s < t->ntaps; ++s) r = std::max(r, std::max(std::abs(t->q1[s]), std::abs(t->q2[s])));
  return r;
}

static ps_status check_table(const ps_grid* g, const ps_table* t) {
  if (!t || t->ntaps < 1 || t->ntaps > PS_MAX_TAPS) return PS_ERR_TABLE;
  const int r = table_radius(t);
  if (r > g->ghost) return PS_ERR_TABLE;
  if (g->bc == PS_BC_DIRICHLET && r > g->ring) return PS_ERR_RADIUS;
  return PS_OK;
}

static ps_status check_grid(const ps_grid* g) {
  if (!g) return PS_ERR_ARG;
  if (g->bc != PS_BC_DIRICHLET && g->bc != PS_BC_PERIODIC) return PS_ERR_ARG;
  if (g->dtype != PS_F64 && g->dtype != PS_F32) return PS_ERR_ARG;
  if (g->arith != PS_ARITH_REF && g->arith != PS_ARITH_NATIVE) return PS_ERR_ARG;
  if (g->rows < 1 || g->cols < 1 || g->rows > (1LL << 30) || g->cols > (1LL << 30))
    return PS_ERR_SHAPE;
  if (g->row0 < 0 || g->row0 + g->rows > g->grows) return PS_ERR_SHAPE;
  return PS_OK;
}

static void fill_gen_table(GenTable& d, const ps_table* t) {
  std::memset(&d, 0, sizeof(d));
  if (!t) return;
  d.ntaps = t->ntaps;
  for (int s = 0; s < t->ntaps; ++s) {
    d.q1[s] = t->q1[s];
    d.q2[s] = t->q2[s];
    d.c[s] = t->c[s];
    d.cf[s] = static_cast<float>(t->c[s]);
  }
}

static dim3 gen_grid(int64_t rows, int64_t cols) {
  const int nsm = std::max(1, dev_info().nsm);
  int64_t gx = (cols + 31) / 32;
  int64_t gy = (rows + 7) / 8;
  gx = std::min<int64_t>(gx, 1024);
  gy = std::min<int64_t>(gy, std::max<int64_t>(1, int64_t(nsm) * 64 / gx + 1));
  gy = std::min<int64_t>(gy, 65535);
  return dim3(unsigned(gx), unsigned(gy));
}

static bool single_slab(const ps_grid* g) { return g->row0 == 0 && g->grows == g->rows; }

// Peer halo targets of a row-slab update (logical-origin pointers of the neighbours'
// u^{k+1} levels; null = no neighbour / exchange done elsewhere).
struct Halo {
  void* up = nullptr;
  void* dn = nullptr;
  int32_t up_rows = 0;
  bool img_consistent = false;  // periodic input images are copies of the core (march)
  bool reverse = false;         // walk tiles bottom-up
};

template <typename T, int A, bool PER, bool FIRST>
static ps_status launch_generic(const ps_grid* g, const void* a, const void* b, void* out,
                                const ps_table* ta, const ps_table* tb, double tau,
                                int64_t rlo, int64_t rhi, cudaStream_t st,
                                const Halo& h = Halo{}) {
  GenParams p;
  std::memset(&p, 0, sizeof(p));
  p.a = at_origin<T>(g, a);
  p.b = at_origin<T>(g, b);
  p.out = at_origin<T>(g, out);
  p.pitch = g->pitch;
  p.rows = int32_t(g->rows);
  p.cols = int32_t(g->cols);
  p.ring = PER ? 0 : g->ring;
  p.radius = std::max(table_radius(ta), tb ? table_radius(tb) : 0);
  p.row0 = int32_t(g->row0);
  p.grows = int32_t(g->grows);
  p.rlo = int32_t(rlo);
  p.rhi = int32_t(rhi);
  p.row_images = (PER && single_slab(g)) ? 1 : 0;
  p.halo_up = h.up;
  p.halo_dn = h.dn;
  p.up_rows = h.up_rows;
  p.tau = tau;
  p.tauf = static_cast<float>(tau);
  fill_gen_table(p.ta, ta);
  fill_gen_table(p.tb, tb);
  if (rhi <= rlo) return PS_OK;
  k_generic<T, A, PER, FIRST><<<gen_grid(rhi - rlo, g->cols), dim3(32, 8), 0, st>>>(p);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return last_cuda_status();
}

template <typename T, int A, class S, bool PER, bool VP = false>
static ps_status launch_stream(const ps_grid* g, const void* uk, const void* ukm1, void* ukp1,
                               const ps_table* t, int64_t rlo, int64_t rhi, cudaStream_t st,
                               const Halo& h, double tau = 0.0) {
  constexpr int NW = PS_NW;
  constexpr int RB = (S::R == 1) ? PS_RB1 : PS_RB2;
  constexpr int NS = PS_NS;
  using Gm = StreamGeom<T, NW, RB, NS>;
  auto kern = k_two_step_stream<T, A, S, PER, NW, RB, NS, VP>;
  static std::once_flag once;
  static int blocks_per_sm = 1;
  std::call_once(once, [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Gm::smem_bytes));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, (NW + 1) * 32,
                                                  Gm::smem_bytes);
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  });
  StreamParams p;
  std::memset(&p, 0, sizeof(p));
  p.uk = at_origin<T>(g, uk);
  p.ukm1 = at_origin<T>(g, ukm1);
  p.ukp1 = at_origin<T>(g, ukp1);
  p.pitch = g->pitch;
  p.rows = int32_t(g->rows);
  p.cols = int32_t(g->cols);
  p.ring = PER ? 0 : g->ring;
  p.row0 = int32_t(g->row0);
  p.grows = int32_t(g->grows);
  p.rlo = int32_t(rlo);
  p.rhi = int32_t(rhi);
  p.row_images = (PER && single_slab(g)) ? 1 : 0;
  p.halo_up = h.up;
  p.halo_dn = h.dn;
  p.up_rows = h.up_rows;
  p.img_exact = h.img_consistent ? 0 : 1;
  p.reverse = h.reverse ? 1 : 0;
  p.tau = tau;
  p.tauf = static_cast<float>(tau);
  for (int s = 0; s < S::N; ++s) {
    p.c[s] = t->c[s];
    p.cf[s] = static_cast<float>(t->c[s]);
  }
  const int64_t nrows = rhi - rlo;
  if (nrows <= 0) return PS_OK;
  const int resident = std::max(1, dev_info().nsm) * blocks_per_sm;
  p.nstrips = int32_t((g->cols + Gm::W - 1) / Gm::W);
  int rc = env_int("PS_ROW_CHUNK", 0);
  if (rc <= 0) {
    // Tiles are claimed dynamically, so balance only needs ~8 tiles per resident block;
    // taller tiles re-read fewer halo rows (2R per tile).  128 rows keeps the tail
    // under one ~25 us tile on the big grids; medium grids drop to >= 16 rows.
    const int64_t want_tiles = int64_t(resident) * 8;
    const int64_t chunks = (want_tiles + p.nstrips - 1) / p.nstrips;
    rc = int(std::max<int64_t>(1, (nrows + chunks - 1) / chunks));
    rc = std::max(rc, std::max(16, 8 * S::R));
    rc = std::min(rc, 128);
    // small grids (L2-resident, latency-bound): more, shorter tiles beat fewer halo rows
    if (p.nstrips * ((nrows + rc - 1) / rc) < resident) rc = std::max(4, 2 * S::R);
  }
  rc = int(std::min<int64_t>(rc, nrows));
  p.rc = rc;
  const int64_t nchunks = (nrows + rc - 1) / rc;
  p.ntiles = int32_t(nchunks * p.nstrips);
  const int grid = int(std::min<int64_t>(p.ntiles, resident));
  const int slot = int(g_launch_seq.fetch_add(1, std::memory_order_relaxed) % kSlots);
  if (launch_pdl(kern, grid, (NW + 1) * 32, Gm::smem_bytes, st, p, slot) != cudaSuccess)
    return PS_ERR_CUDA;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return last_cuda_status();
}

template <typename T, int A, bool PER>
static ps_status dispatch_two_step(const ps_grid* g, const void* uk, const void* ukm1, void* ukp1,
                                   const ps_table* t, int64_t lo, int64_t hi, cudaStream_t st,
                                   const Halo& h) {
  // The streaming kernel wants >= 4 rows/cols and at least one wrap (n >= R) for images.
  const bool small = g->rows < 4 || g->cols < 4;
  if (!small && env_int("PS_FORCE_GENERIC", 0) == 0) {
    if (shape_matches<ShapeP5>(t))
      return launch_stream<T, A, ShapeP5, PER>(g, uk, ukm1, ukp1, t, lo, hi, st, h);
    if (shape_matches<ShapeP9>(t))
      return launch_stream<T, A, ShapeP9, PER>(g, uk, ukm1, ukp1, t, lo, hi, st, h);
    if (shape_matches<ShapeC9>(t))
      return launch_stream<T, A, ShapeC9, PER>(g, uk, ukm1, ukp1, t, lo, hi, st, h);
    if (shape_matches<ShapeP13>(t))
      return launch_stream<T, A, ShapeP13, PER>(g, uk, ukm1, ukp1, t, lo, hi, st, h);
  }
  return launch_generic<T, A, PER, false>(g, uk, ukm1, ukp1, t, nullptr, 0.0, lo, hi, st, h);
}

template <typename T, int A>
static ps_status dispatch_two_step_bc(const ps_grid* g, const void* uk, const void* ukm1,
                                      void* ukp1, const ps_table* t, int64_t lo, int64_t hi,
                                      cudaStream_t st, const Halo& h) {
  if (g->bc == PS_BC_PERIODIC)
    return dispatch_two_step<T, A, true>(g, uk, ukm1, ukp1, t, lo, hi, st, h);
  return dispatch_two_step<T, A, false>(g, uk, ukm1, ukp1, t, lo, hi, st, h);
}

static ps_status two_step_impl(const ps_grid* g, const void* uk, const void* ukm1, void* ukp1,
                               const ps_table* t, int64_t lo, int64_t hi, cudaStream_t st,
                               const Halo& h = Halo{}) {
  if (g->dtype == PS_F64)
    return dispatch_two_step_bc<double, ARITH_REF>(g, uk, ukm1, ukp1, t, lo, hi, st, h);
  if (g->arith == PS_ARITH_NATIVE)
    return dispatch_two_step_bc<float, ARITH_NATIVE>(g, uk, ukm1, ukp1, t, lo, hi, st, h);
  return dispatch_two_step_bc<float, ARITH_REF>(g, uk, ukm1, ukp1, t, lo, hi, st, h);
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Inside a march every periodic level was produced by this library (images = core copies);
// odd steps walk their tiles bottom-up so they start on the rows the previous step wrote
// last, which grids of a few hundred MB still find in the 126 MB L2.
static bool alternate_walk(const ps_grid* g) {
  // only grids whose level is within ~2x the L2 keep useful rows between launches
  // (measured: +4 % on C2's 134 MB levels; on 17 GB levels the reversed walk cost 6 %)
  static const int mode = env_int("PS_ALTERNATE", -1);
  if (mode >= 0) return mode != 0;
  return ps_level_bytes(g) <= (size_t(256) << 20);
}

static Halo march_opts(const ps_grid* g, int64_t k) {
  Halo h;
  h.img_consistent = true;
  h.reverse = (k & 1) != 0 && alternate_walk(g);
  return h;
}

// ---------------------------------------------------------------------------
// Temporal blocking (ps_tblock.cuh)
// ---------------------------------------------------------------------------
// Geometry (measured on B200, profiles/ and DESIGN.md): 4 consumer warps x 3 stages,
// except f32 at depth 4, whose ~224-register windows allow one block per SM — there 8
// warps x 2 stages keep more warps resident.  Tuning builds override with -D.
#ifndef PS_TB_NW
#define PS_TB_NW 0
#endif
#ifndef PS_TB_RB
#define PS_TB_RB 0  // 0: 2R+1 rows per stage, so a stage is one full window rotation
#endif
#ifndef PS_TB_NS
#define PS_TB_NS 0
#endif
template <typename T, int TS>
constexpr int tb_nw() {
  return PS_TB_NW > 0 ? PS_TB_NW : ((TS == 4 && sizeof(T) == 4) ? 8 : 4);
}
template <typename T, int TS>
constexpr int tb_ns() {
  return PS_TB_NS > 0 ? PS_TB_NS : ((TS == 4 && sizeof(T) == 4) ? 2 : 3);
}

template <typename T, int A, class S, int TS, bool PER>
static ps_status launch_tb(const ps_grid* g, const void* uk, const void* ukm1, void* out_prev,
                           void* out_last, const ps_table* t, int64_t rlo, int64_t rhi,
                           cudaStream_t st, bool reverse) {
  constexpr int NW = tb_nw<T, TS>(), NS = tb_ns<T, TS>();
  constexpr int RB = PS_TB_RB > 0 ? PS_TB_RB : 2 * S::R + 1;
  using Gm = TBGeom<T, NW, RB, NS, S::R, TS>;
  auto kern = k_two_step_tb<T, A, S, TS, PER, NW, RB, NS>;
  static std::once_flag once;
  static int blocks_per_sm = 1;
  std::call_once(once, [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Gm::smem_bytes));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, (NW + 1) * 32,
                                                  Gm::smem_bytes);
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  });
  const int64_t nrows = rhi - rlo;
  if (nrows <= 0) return PS_OK;
  TBParams p;
  std::memset(&p, 0, sizeof(p));
  p.uk = at_origin<T>(g, uk);
  p.ukm1 = at_origin<T>(g, ukm1);
  p.out_prev = at_origin<T>(g, out_prev);
  p.out_last = at_origin<T>(g, out_last);
  p.pitch = g->pitch;
  p.rows = int32_t(g->rows);
  p.cols = int32_t(g->cols);
  p.ring = PER ? 0 : g->ring;
  p.row0 = int32_t(g->row0);
  p.grows = int32_t(g->grows);
  p.rlo = int32_t(rlo);
  p.rhi = int32_t(rhi);
  p.gmin = -int32_t(g->ghost);
  p.gmax = int32_t(g->rows + g->ghost);
  p.cmax = int32_t(g->pitch - (g->origin - g->ghost * g->pitch));
  p.reverse = reverse ? 1 : 0;
  for (int s = 0; s < S::N; ++s) {
    p.c[s] = t->c[s];
    p.cf[s] = static_cast<float>(t->c[s]);
  }
  const int resident = std::max(1, dev_info().nsm) * blocks_per_sm;
  p.nstrips = int32_t((g->cols + Gm::W - 1) / Gm::W);
  int rc = env_int("PS_TB_ROW_CHUNK", 0);
  if (rc <= 0) {
    const int64_t want_tiles = int64_t(resident) * 8;
    const int64_t chunks = (want_tiles + p.nstrips - 1) / p.nstrips;
    rc = int(std::max<int64_t>(1, (nrows + chunks - 1) / chunks));
    rc = std::max(rc, std::max(32, 8 * S::R * TS));
    rc = std::min(rc, 256);
  }
  rc = int(std::min<int64_t>(rc, nrows));
  p.rc = rc;
  p.ntiles = int32_t(((nrows + rc - 1) / rc) * p.nstrips);
  const int grid = int(std::min<int64_t>(p.ntiles, resident));
  const int slot = int(g_launch_seq.fetch_add(1, std::memory_order_relaxed) % kSlots);
  if (launch_pdl(kern, grid, (NW + 1) * 32, Gm::smem_bytes, st, p, slot) != cudaSuccess)
    return PS_ERR_CUDA;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return last_cuda_status();
}

template <typename T, int A, int TS>
static ps_status dispatch_tb(const ps_grid* g, const void* uk, const void* ukm1, void* op,
                             void* ol, const ps_table* t, int64_t lo, int64_t hi,
                             cudaStream_t st, bool rev) {
  if (shape_matches<ShapeP5>(t))
    return g->bc == PS_BC_PERIODIC ? launch_tb<T, A, ShapeP5, TS, true>(g, uk, ukm1, op, ol, t, lo, hi, st, rev) : launch_tb<T, A, ShapeP5, TS, false>(g, uk, ukm1, op, ol, t, lo, hi, st, rev);
  if (shape_matches<ShapeP9>(t))
    return g->bc == PS_BC_PERIODIC ? launch_tb<T, A, ShapeP9, TS, true>(g, uk, ukm1, op, ol, t, lo, hi, st, rev) : launch_tb<T, A, ShapeP9, TS, false>(g, uk, ukm1, op, ol, t, lo, hi, st, rev);
  if (shape_matches<ShapeC9>(t))
    return g->bc == PS_BC_PERIODIC ? launch_tb<T, A, ShapeC9, TS, true>(g, uk, ukm1, op, ol, t, lo, hi, st, rev) : launch_tb<T, A, ShapeC9, TS, false>(g, uk, ukm1, op, ol, t, lo, hi, st, rev);
  if (shape_matches<ShapeP13>(t))
    return g->bc == PS_BC_PERIODIC ? launch_tb<T, A, ShapeP13, TS, true>(g, uk, ukm1, op, ol, t, lo, hi, st, rev) : launch_tb<T, A, ShapeP13, TS, false>(g, uk, ukm1, op, ol, t, lo, hi, st, rev);
  return PS_ERR_TABLE;
}

template <int TS>
static ps_status tb_impl(const ps_grid* g, const void* uk, const void* ukm1, void* op, void* ol,
                         const ps_table* t, int64_t lo, int64_t hi, cudaStream_t st, bool rev) {
  if (g->dtype == PS_F64)
    return dispatch_tb<double, ARITH_REF, TS>(g, uk, ukm1, op, ol, t, lo, hi, st, rev);
  if (g->arith == PS_ARITH_NATIVE)
    return dispatch_tb<float, ARITH_NATIVE, TS>(g, uk, ukm1, op, ol, t, lo, hi, st, rev);
  return dispatch_tb<float, ARITH_REF, TS>(g, uk, ukm1, op, ol, t, lo, hi, st, rev);
}

static ps_status two_step_tb_impl(const ps_grid* g, const void* uk, const void* ukm1, void* op,
                                  void* ol, const ps_table* t, int tsteps, cudaStream_t st,
                                  int64_t lo = 0, int64_t hi = -1, bool rev = false) {
  if (hi < 0) hi = g->rows;
  switch (tsteps) {
    case 2: return tb_impl<2>(g, uk, ukm1, op, ol, t, lo, hi, st, rev);
    case 4: return tb_impl<4>(g, uk, ukm1, op, ol, t, lo, hi, st, rev);
    default: return PS_ERR_ARG;
  }
}

static bool tb_supported(const ps_grid* g, const ps_table* t, int tsteps) {
  const bool shape = shape_matches<ShapeP5>(t) || shape_matches<ShapeP9>(t) ||
                     shape_matches<ShapeC9>(t) || shape_matches<ShapeP13>(t);
  if (!shape || g->rows < 4 || g->cols < 4) return false;
  if (g->bc == PS_BC_DIRICHLET) return true;
  // periodic: single slab, images to depth R*tsteps must fit the ghost band, and one
  // wrap must cover them
  const int64_t D = int64_t(table_radius(t)) * tsteps;
  return single_slab(g) && D <= g->ghost && D <= g->rows && D <= g->cols;
}

// ---------------------------------------------------------------------------
// CUDA-graph replay of the march: six launches (two level-rotation cycles, so the
// alternating tile direction lines up too) are captured once per (grid, levels, table,
// phase) and replayed nsteps/6 times, which removes per-launch CPU cost and launch gaps
// on latency-bound grids.
// ---------------------------------------------------------------------------
constexpr int kGraphCycle = 6;
struct GraphKey {
  ps_grid g;
  void* lvl[3];
  int32_t cur;
  int32_t dev;
  ps_table t;
};
struct GraphEntry {
  GraphKey key;
  cudaGraphExec_t exec;
};
static std::mutex g_graph_mu;
static GraphEntry g_graphs[32];
static int g_ngraphs = 0;
static int g_graph_next = 0;

static cudaStream_t capture_stream(int dev) {
  static cudaStream_t streams[64] = {};
  if (dev < 0 || dev >= 64) return nullptr;
  if (!streams[dev]) cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking);
  return streams[dev];
}

static cudaGraphExec_t cycle_graph(const ps_grid* g, void* lvl[3], int cur, const ps_table* t) {
  GraphKey key;
  std::memset(&key, 0, sizeof(key));
  key.g = *g;
  for (int x = 0; x < 3; ++x) key.lvl[x] = lvl[x];
  key.cur = cur;
  cudaGetDevice(&key.dev);
  key.t.ntaps = t->ntaps;
  for (int s = 0; s < t->ntaps; ++s) {
    key.t.q1[s] = t->q1[s];
    key.t.q2[s] = t->q2[s];
    key.t.c[s] = t->c[s];
  }
  std::lock_guard<std::mutex> lk(g_graph_mu);
  for (int e = 0; e < g_ngraphs; ++e)
    if (std::memcmp(&g_graphs[e].key, &key, sizeof(key)) == 0) return g_graphs[e].exec;
  cudaStream_t cs = capture_stream(key.dev);
  if (!cs) return nullptr;
  if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  int c = cur;
  ps_status st = PS_OK;
  for (int k = 0; k < kGraphCycle && st == PS_OK; ++k) {
    st = two_step_impl(g, lvl[c], lvl[(c + 2) % 3], lvl[(c + 1) % 3], t, 0, g->rows, cs,
                       march_opts(g, k));
    c = (c + 1) % 3;
  }
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(cs, &graph);
  cudaGraphExec_t exec = nullptr;
  if (st != PS_OK || ec != cudaSuccess || !graph ||
      cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    return nullptr;
  }
  cudaGraphDestroy(graph);
  g_launches.fetch_sub(kGraphCycle, std::memory_order_relaxed);  // captured, not executed
  GraphEntry& slot = g_graphs[g_graph_next];
  if (g_graph_next < g_ngraphs && slot.exec) cudaGraphExecDestroy(slot.exec);
  slot.key = key;
  slot.exec = exec;
  g_graph_next = (g_graph_next + 1) % 32;
  g_ngraphs = std::min(g_ngraphs + 1, 32);
  return exec;
}

// First step as two streaming launches: u1 <- -fl(tau * A_v(v0)) (VP), then the ordinary
// two-step kernel u1 <- fl(A_u(u0) - u1) = fl(A_u(u0) + fl(tau * A_v(v0))), bit for bit the
// reference's first step.  Both tables must have a specialised shape.
template <typename T, int A, bool PER>
static ps_status first_step_stream(const ps_grid* g, const void* u0, const void* v0, void* u1,
                                   const ps_table* tu, const ps_table* tv, double tau,
                                   cudaStream_t st, bool* done) {
  *done = true;
  const Halo h;
  ps_status s;
  if (shape_matches<ShapeP5>(tv))
    s = launch_stream<T, A, ShapeP5, PER, true>(g, v0, v0, u1, tv, 0, g->rows, st, h, tau);
  else if (shape_matches<ShapeP9>(tv))
    s = launch_stream<T, A, ShapeP9, PER, true>(g, v0, v0, u1, tv, 0, g->rows, st, h, tau);
  else if (shape_matches<ShapeC9>(tv))
    s = launch_stream<T, A, ShapeC9, PER, true>(g, v0, v0, u1, tv, 0, g->rows, st, h, tau);
  else if (shape_matches<ShapeP13>(tv))
    s = launch_stream<T, A, ShapeP13, PER, true>(g, v0, v0, u1, tv, 0, g->rows, st, h, tau);
  else {
    *done = false;
    return PS_OK;
  }
  if (s != PS_OK) return s;
  return dispatch_two_step<T, A, PER>(g, u0, u1, u1, tu, 0, g->rows, st, h);
}

static bool stream_shape(const ps_table* t) {
  return shape_matches<ShapeP5>(t) || shape_matches<ShapeP9>(t) || shape_matches<ShapeC9>(t) ||
         shape_matches<ShapeP13>(t);
}

}  // namespace ps

// ===========================================================================
// C-ABI
// ===========================================================================
using namespace ps;

extern "C" {

ps_status ps_layout_init(ps_grid* g, int64_t rows, int64_t cols, int32_t ghost, int32_t ring,
                         int32_t bc, int32_t dtype, int32_t arith) {
  if (!g) return PS_ERR_ARG;
  if (bc != PS_BC_DIRICHLET && bc != PS_BC_PERIODIC) return PS_ERR_ARG;
  if (dtype != PS_F64 && dtype != PS_F32) return PS_ERR_ARG;
  if (arith != PS_ARITH_REF && arith != PS_ARITH_NATIVE) return PS_ERR_ARG;
  if (rows < 1 || cols < 1 || rows > (1LL << 30) || cols > (1LL << 30)) return PS_ERR_SHAPE;
  if (ghost < 0 || ghost > PS_MAX_GHOST) return PS_ERR_ARG;
  if (bc == PS_BC_DIRICHLET && (ring < 0 || 2 * int64_t(ring) > std::min(rows, cols)))
    return PS_ERR_SHAPE;
  const int64_t esz = dtype == PS_F64 ? 8 : 4;
  const int64_t line = 128 / esz;             // elements per 128-byte line
  const int64_t G = std::max<int64_t>(2, ghost);
  const int64_t cpad = ((G + line - 1) / line) * line;  // left pad, keeps (0,0) 128-B aligned
  // right side: strip overrun of the streaming kernel (whole 16-byte vector + halo
  // vector) and the periodic images, rounded to a 128-byte multiple.
  const int64_t vec = 16 / esz;
  const int64_t right = std::max<int64_t>(G, 2 * vec);
  int64_t pitch = cpad + ((cols + vec - 1) / vec) * vec + right;
  pitch = ((pitch + line - 1) / line) * line;
  g->rows = rows;
  g->cols = cols;
  g->pitch = pitch;
  g->ghost = G;
  g->origin = G * pitch + cpad;
  g->row0 = 0;
  g->grows = rows;
  g->ring = bc == PS_BC_DIRICHLET ? ring : 0;
  g->bc = bc;
  g->dtype = dtype;
  g->arith = dtype == PS_F64 ? PS_ARITH_REF : arith;
  return PS_OK;
}

ps_status ps_slab_layout_init(ps_grid* g, int64_t grows, int64_t cols, int64_t row0,
                              int64_t rows, int32_t ghost, int32_t ring, int32_t bc,
                              int32_t dtype, int32_t arith) {
  if (row0 < 0 || rows < 1 || row0 + rows > grows) return PS_ERR_SHAPE;
  ps_status s = ps_layout_init(g, grows, cols, ghost, ring, bc, dtype, arith);
  if (s != PS_OK) return s;
  g->rows = rows;
  g->row0 = row0;
  g->grows = grows;
  return PS_OK;
}

size_t ps_level_bytes(const ps_grid* g) {
  if (!g) return 0;
  const size_t esz = g->dtype == PS_F64 ? 8 : 4;
  return size_t(g->rows + 2 * g->ghost) * size_t(g->pitch) * esz;
}

void* ps_level_alloc(const ps_grid* g) {
  const size_t bytes = ps_level_bytes(g);
  if (!bytes) return nullptr;
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
  if (cudaMemset(p, 0, bytes) != cudaSuccess) {
    cudaFree(p);
    return nullptr;
  }
  return p;
}

void ps_level_free(void* level) {
  if (level) cudaFree(level);
}

static ps_status copy_block(const ps_grid* g, void* level, const void* host, int64_t rows_h,
                            int64_t cols_h, int64_t hpitch, int32_t kind, void* stream,
                            bool in) {
  ps_status s = check_grid(g);
  if (s != PS_OK) return s;
  if (!level || !host || rows_h < 0 || cols_h < 0 || hpitch < cols_h) return PS_ERR_ARG;
  if (kind < 0 || kind > 4) return PS_ERR_ARG;
  const int64_t extra = g->bc == PS_BC_PERIODIC ? g->ghost : 0;
  if (rows_h > g->rows + extra || cols_h > g->cols + extra) return PS_ERR_SHAPE;
  if (rows_h == 0 || cols_h == 0) return PS_OK;
  const size_t esz = g->dtype == PS_F64 ? 8 : 4;
  char* dev = static_cast<char*>(level) + g->origin * esz;
  cudaError_t e;
  if (in)
    e = cudaMemcpy2DAsync(dev, g->pitch * esz, host, hpitch * esz, cols_h * esz, rows_h,
                          cudaMemcpyKind(kind), static_cast<cudaStream_t>(stream));
  else
    e = cudaMemcpy2DAsync(const_cast<void*>(host), hpitch * esz, dev, g->pitch * esz,
                          cols_h * esz, rows_h, cudaMemcpyKind(kind),
                          static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? PS_OK : PS_ERR_CUDA;
}

ps_status ps_copy_in(const ps_grid* g, void* level, const void* src, int64_t rows_h,
                     int64_t cols_h, int64_t src_pitch, int32_t kind, void* stream) {
  return copy_block(g, level, src, rows_h, cols_h, src_pitch, kind, stream, true);
}

ps_status ps_copy_out(const ps_grid* g, const void* level, void* dst, int64_t rows_h,
                      int64_t cols_h, int64_t dst_pitch, int32_t kind, void* stream) {
  return copy_block(g, const_cast<void*>(level), dst, rows_h, cols_h, dst_pitch, kind, stream,
                    false);
}

ps_status ps_fill_ghosts(const ps_grid* g, void* level, int32_t keep_alias, void* stream) {
  ps_status s = check_grid(g);
  if (s != PS_OK) return s;
  if (!level) return PS_ERR_ARG;
  if (g->bc != PS_BC_PERIODIC) return PS_OK;
  const int64_t total = 2 * g->ghost * (g->cols + 2 * g->ghost) + 2 * g->ghost * g->rows;
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((total + threads - 1) / threads, 65535);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (g->dtype == PS_F64)
    k_fill_ghosts<double><<<unsigned(blocks), threads, 0, st>>>(
        at_origin<double>(g, level), g->pitch, int32_t(g->rows), int32_t(g->cols),
        int32_t(g->ghost), keep_alias);
  else
    k_fill_ghosts<float><<<unsigned(blocks), threads, 0, st>>>(
        at_origin<float>(g, level), g->pitch, int32_t(g->rows), int32_t(g->cols),
        int32_t(g->ghost), keep_alias);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return last_cuda_status();
}

ps_status ps_first_step(const ps_grid* g, const void* u0, const void* v0, void* u1,
                        const ps_table* tu, const ps_table* tv, double tau, void* stream) {
  ps_status s = check_grid(g);
  if (s != PS_OK) return s;
  if (!u0 || !v0 || !u1) return PS_ERR_ARG;
  if ((s = check_table(g, tu)) != PS_OK) return s;
  if ((s = check_table(g, tv)) != PS_OK) return s;
  if (!aligned16(u0) || !aligned16(v0) || !aligned16(u1)) return PS_ERR_ALIGN;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool per = g->bc == PS_BC_PERIODIC;
  if (u1 != u0 && u1 != v0 && stream_shape(tu) && stream_shape(tv) && g->rows >= 4 &&
      g->cols >= 4 && env_int("PS_FORCE_GENERIC", 0) == 0) {
    bool done = false;
    if (g->dtype == PS_F64)
      s = per ? first_step_stream<double, ARITH_REF, true>(g, u0, v0, u1, tu, tv, tau, st, &done)
              : first_step_stream<double, ARITH_REF, false>(g, u0, v0, u1, tu, tv, tau, st, &done);
    else if (g->arith == PS_ARITH_NATIVE)
      s = per ? first_step_stream<float, ARITH_NATIVE, true>(g, u0, v0, u1, tu, tv, tau, st, &done)
              : first_step_stream<float, ARITH_NATIVE, false>(g, u0, v0, u1, tu, tv, tau, st,
                                                              &done);
    else
      s = per ? first_step_stream<float, ARITH_REF, true>(g, u0, v0, u1, tu, tv, tau, st, &done)
              : first_step_stream<float, ARITH_REF, false>(g, u0, v0, u1, tu, tv, tau, st, &done);
    if (done || s != PS_OK) return s;
  }
  if (g->dtype == PS_F64)
    return per ? launch_generic<double, ARITH_REF, true, true>(g, u0, v0, u1, tu, tv, tau, 0, g->rows, st)
               : launch_generic<double, ARITH_REF, false, true>(g, u0, v0, u1, tu, tv, tau, 0, g->rows, st);
  if (g->arith == PS_ARITH_NATIVE)
    return per ? launch_generic<float, ARITH_NATIVE, true, true>(g, u0, v0, u1, tu, tv, tau, 0, g->rows, st)
               : launch_generic<float, ARITH_NATIVE, false, true>(g, u0, v0, u1, tu, tv, tau, 0, g->rows, st);
  return per ? launch_generic<float, ARITH_REF, true, true>(g, u0, v0, u1, tu, tv, tau, 0, g->rows, st)
             : launch_generic<float, ARITH_REF, false, true>(g, u0, v0, u1, tu, tv, tau, 0, g->rows, st);
}

ps_status ps_two_step(const ps_grid* g, const void* uk, const void* ukm1, void* ukp1,
                      const ps_table* t, void* stream) {
  ps_status s = check_grid(g);
  if (s != PS_OK) return s;
  if (!uk || !ukm1 || !ukp1 || ukp1 == uk) return PS_ERR_ARG;
  if ((s = check_table(g, t)) != PS_OK) return s;
  if (!aligned16(uk) || !aligned16(ukm1) || !aligned16(ukp1)) return PS_ERR_ALIGN;
  return two_step_impl(g, uk, ukm1, ukp1, t, 0, g->rows, static_cast<cudaStream_t>(stream));
}

ps_status ps_two_step_rows(const ps_grid* g, const void* uk, const void* ukm1, void* ukp1,
                           const ps_table* t, int64_t row_lo, int64_t row_hi, void* stream) {
  ps_status s = check_grid(g);
  if (s != PS_OK) return s;
  if (!uk || !ukm1 || !ukp1 || ukp1 == uk) return PS_ERR_ARG;
  if (row_lo < 0 || row_hi > g->rows || row_lo > row_hi) return PS_ERR_ARG;
  if ((s = check_table(g, t)) != PS_OK) return s;
  if (!aligned16(uk) || !aligned16(ukm1) || !aligned16(ukp1)) return PS_ERR_ALIGN;
  return two_step_impl(g, uk, ukm1, ukp1, t, row_lo, row_hi, static_cast<cudaStream_t>(stream));
}

ps_status ps_two_step_halo(const ps_grid* g, const void* uk, const void* ukm1, void* ukp1,
                           const ps_table* t, int64_t row_lo, int64_t row_hi, void* up_ukp1,
                           int64_t up_rows, void* dn_ukp1, void* stream) {
  ps_status s = check_grid(g);
  if (s != PS_OK) return s;
  if (!uk || !ukm1 || !ukp1 || ukp1 == uk) return PS_ERR_ARG;
  if (row_lo < 0 || row_hi > g->rows || row_lo > row_hi) return PS_ERR_ARG;
  if (g->bc != PS_BC_DIRICHLET) return PS_ERR_ARG;
  if ((s = check_table(g, t)) != PS_OK) return s;
  if (up_ukp1 && (up_rows < table_radius(t) || !aligned16(up_ukp1))) return PS_ERR_ARG;
  if (dn_ukp1 && !aligned16(dn_ukp1)) return PS_ERR_ALIGN;
  if (table_radius(t) > g->rows) return PS_ERR_SHAPE;
  if (!aligned16(uk) || !aligned16(ukm1) || !aligned16(ukp1)) return PS_ERR_ALIGN;
  const size_t esz = g->dtype == PS_F64 ? 8 : 4;
  Halo h;
  h.up = up_ukp1 ? static_cast<char*>(up_ukp1) + g->origin * esz : nullptr;
  h.dn = dn_ukp1 ? static_cast<char*>(dn_ukp1) + g->origin * esz : nullptr;
  h.up_rows = int32_t(up_rows);
  return two_step_impl(g, uk, ukm1, ukp1, t, row_lo, row_hi, static_cast<cudaStream_t>(stream),
                       h);
}

ps_status ps_ipc_get_handle(const void* dev_ptr, void* handle64, int64_t* offset) {
  if (!dev_ptr || !handle64 || !offset) return PS_ERR_ARG;
  // IPC handles name whole allocations; a pointer from a caching allocator may sit
  // inside a larger block, so report its offset from the allocation base.
  // (driver entry point fetched at run time: libps.so must load on hosts without a driver)
  using AddrRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static AddrRangeFn addr_range = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<AddrRangeFn>(fn);
  }();
  if (!addr_range) return PS_ERR_CUDA;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (addr_range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return PS_ERR_CUDA;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)) != cudaSuccess) return PS_ERR_CUDA;
  std::memcpy(handle64, &h, sizeof(h));
  *offset = int64_t(reinterpret_cast<uintptr_t>(dev_ptr) - uintptr_t(base));
  return PS_OK;
}

ps_status ps_ipc_open(const void* handle64, void** dev_ptr) {
  if (!handle64 || !dev_ptr) return PS_ERR_ARG;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  if (cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
    return PS_ERR_CUDA;
  return PS_OK;
}

ps_status ps_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return PS_ERR_ARG;
  return cudaIpcCloseMemHandle(dev_ptr) == cudaSuccess ? PS_OK : PS_ERR_CUDA;
}

ps_status ps_march(const ps_grid* g, void* lvl[3], int64_t nsteps, const ps_table* t,
                   int32_t* newest, void* stream) {
  ps_status s = check_grid(g);
  if (s != PS_OK) return s;
  if (!lvl || !newest || nsteps < 0 || *newest < 0 || *newest > 2) return PS_ERR_ARG;
  if (!lvl[0] || !lvl[1] || !lvl[2]) return PS_ERR_ARG;
  if ((s = check_table(g, t)) != PS_OK) return s;
  for (int x = 0; x < 3; ++x)
    if (!aligned16(lvl[x])) return PS_ERR_ALIGN;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int cur = *newest;
  int64_t k = 0;
  if (nsteps >= 2 * kGraphCycle && env_int("PS_GRAPH", 1) != 0) {
    if (cudaGraphExec_t exec = cycle_graph(g, lvl, cur, t)) {
      for (; k + kGraphCycle <= nsteps; k += kGraphCycle) {
        if (cudaGraphLaunch(exec, st) != cudaSuccess) return PS_ERR_CUDA;
        g_launches.fetch_add(kGraphCycle, std::memory_order_relaxed);
      }
      // whole rotation cycles return the levels to the same phase: cur is unchanged
    }
  }
  for (; k < nsteps; ++k) {
    const int prev = (cur + 2) % 3;
    const int next = (cur + 1) % 3;
    if ((s = two_step_impl(g, lvl[cur], lvl[prev], lvl[next], t, 0, g->rows, st,
                           march_opts(g, k))) != PS_OK)
      return s;
    cur = next;
  }
  *newest = cur;
  return PS_OK;
}

ps_status ps_two_step_tb(const ps_grid* g, const void* uk, const void* ukm1, void* out_prev,
                         void* out_last, const ps_table* t, int32_t tsteps, void* stream) {
  ps_status s = check_grid(g);
  if (s != PS_OK) return s;
  if (!uk || !ukm1 || !out_prev || !out_last) return PS_ERR_ARG;
  if (out_prev == uk || out_prev == ukm1 || out_last == uk || out_last == ukm1 ||
      out_prev == out_last)
    return PS_ERR_ARG;
  if ((s = check_table(g, t)) != PS_OK) return s;
  if (!tb_supported(g, t, tsteps)) return PS_ERR_ARG;
  if (!aligned16(uk) || !aligned16(ukm1) || !aligned16(out_prev) || !aligned16(out_last))
    return PS_ERR_ALIGN;
  return two_step_tb_impl(g, uk, ukm1, out_prev, out_last, t, tsteps,
                          static_cast<cudaStream_t>(stream));
}

ps_status ps_two_step_tb_rows(const ps_grid* g, const void* uk, const void* ukm1,
                              void* out_prev, void* out_last, const ps_table* t, int32_t tsteps,
                              int64_t row_lo, int64_t row_hi, void* stream) {
  ps_status s = check_grid(g);
  if (s != PS_OK) return s;
  if (!uk || !ukm1 || !out_prev || !out_last) return PS_ERR_ARG;
  if (out_prev == uk || out_prev == ukm1 || out_last == uk || out_last == ukm1 ||
      out_prev == out_last)
    return PS_ERR_ARG;
  if (row_lo < 0 || row_hi > g->rows || row_lo > row_hi) return PS_ERR_ARG;
  if ((s = check_table(g, t)) != PS_OK) return s;
  if (!tb_supported(g, t, tsteps)) return PS_ERR_ARG;
  // the fused pass reads R*tsteps halo rows of u^k beyond the launch's row range
  if (int64_t(table_radius(t)) * tsteps > g->ghost && !single_slab(g)) return PS_ERR_SHAPE;
  if (!aligned16(uk) || !aligned16(ukm1) || !aligned16(out_prev) || !aligned16(out_last))
    return PS_ERR_ALIGN;
  return two_step_tb_impl(g, uk, ukm1, out_prev, out_last, t, tsteps,
                          static_cast<cudaStream_t>(stream), row_lo, row_hi);
}

ps_status ps_march_tb(const ps_grid* g, void* lvl[4], int64_t nsteps, const ps_table* t,
                      int32_t tsteps, int32_t* newest, int32_t* previous, void* stream) {
  ps_status s = check_grid(g);
  if (s != PS_OK) return s;
  if (!lvl || !newest || !previous || nsteps < 0) return PS_ERR_ARG;
  int cur = *newest, prev = *previous;
  if (cur < 0 || cur > 3 || prev < 0 || prev > 3 || cur == prev) return PS_ERR_ARG;
  for (int x = 0; x < 4; ++x)
    if (!lvl[x] || !aligned16(lvl[x])) return lvl[x] ? PS_ERR_ALIGN : PS_ERR_ARG;
  if ((s = check_table(g, t)) != PS_OK) return s;
  if (tsteps != 1 && tsteps != 2 && tsteps != 4) return PS_ERR_ARG;
  if (tsteps > 1 && !tb_supported(g, t, tsteps)) return PS_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t k = 0;
  if (tsteps > 1 && g->bc == PS_BC_PERIODIC && nsteps >= tsteps) {
    // blocked passes read wrap-around images to depth R*tsteps; levels written by a
    // single step (first step, earlier remainders) carry them only to depth R
    if ((s = ps_fill_ghosts(g, lvl[cur], 0, stream)) != PS_OK) return s;
    if ((s = ps_fill_ghosts(g, lvl[prev], 0, stream)) != PS_OK) return s;
  }
  auto free_pair = [&](int a, int b, int* f1, int* f2) {
    int n = 0;
    for (int x = 0; x < 4; ++x)
      if (x != a && x != b) (n++ == 0 ? *f1 : *f2) = x;
  };
  if (tsteps > 1) {
    const bool alternate = alternate_walk(g);
    for (int64_t blk = 0; k + tsteps <= nsteps; k += tsteps, ++blk) {
      int f1, f2;
      free_pair(cur, prev, &f1, &f2);
      if ((s = two_step_tb_impl(g, lvl[cur], lvl[prev], lvl[f1], lvl[f2], t, tsteps, st, 0,
                                g->rows, alternate && (blk & 1))) != PS_OK)
        return s;
      prev = f1;
      cur = f2;
    }
  }
  for (; k < nsteps; ++k) {
    int f1, f2;
    free_pair(cur, prev, &f1, &f2);
    if ((s = two_step_impl(g, lvl[cur], lvl[prev], lvl[f1], t, 0, g->rows, st)) != PS_OK) return s;
    prev = cur;
    cur = f1;
  }
  *newest = cur;
  *previous = prev;
  return PS_OK;
}

ps_status ps_gaussian_sum(const ps_grid* g, void* level, int32_t K, const double* cx,
                          const double* cy, const double* width, const double* amp, int64_t n,
                          void* stream) {
  ps_status s = check_grid(g);
  if (s != PS_OK) return s;
  if (!level || K < 0 || K > kMaxGauss || n < 1) return PS_ERR_ARG;
  if (K > 0 && (!cx || !cy || !width || !amp)) return PS_ERR_ARG;
  static thread_local GaussParams p;
  p.K = K;
  p.rows = int32_t(g->rows);
  p.cols = int32_t(g->cols);
  p.row0 = int32_t(g->row0);
  p.pitch = g->pitch;
  p.n = double(n);
  for (int k = 0; k < K; ++k) {
    p.cx[k] = cx[k];
    p.cy[k] = cy[k];
    p.w2[k] = 2.0 * (width[k] * width[k]);
    p.amp[k] = amp[k];
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const dim3 grid = gen_grid(g->rows, g->cols);
  if (g->dtype == PS_F64)
    k_gaussian<double><<<grid, dim3(32, 8), 0, st>>>(p, at_origin<double>(g, level));
  else
    k_gaussian<float><<<grid, dim3(32, 8), 0, st>>>(p, at_origin<float>(g, level));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if ((s = last_cuda_status()) != PS_OK) return s;
  return ps_fill_ghosts(g, level, 0, stream);
}

struct ps_errsum {
  ps::ErrsumPlan plan;
};

ps_errsum* ps_errsum_create(int64_t rows_h, int64_t cols_h) {
  if (rows_h < 1 || cols_h < 1) return nullptr;
  const int64_t N = rows_h * cols_h;
  struct Ref {
    bool leaf;
    int32_t idx;
  };
  struct Internal {
    Ref l, r;
    int32_t height;
  };
  std::vector<int64_t> ls;
  std::vector<int32_t> ll;
  std::vector<Internal> ints;
  // numpy's pairwise order: ranges <= 128 are leaves, larger ones split at n/2 rounded
  // down to a multiple of 8 (explicit stack instead of recursion).
  struct Frame {
    int64_t start, n;
    int state;
    Ref left;
    int32_t hl;
  };
  std::vector<Frame> stack;
  stack.push_back({0, N, 0, {true, 0}, 0});
  Ref ret{true, 0};
  int32_t ret_h = 0;
  while (!stack.empty()) {
    Frame& f = stack.back();
    if (f.n <= ps::kPwBlock) {
      ls.push_back(f.start);
      ll.push_back(int32_t(f.n));
      ret = {true, int32_t(ls.size() - 1)};
      ret_h = 0;
      stack.pop_back();
      continue;
    }
    int64_t n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.state == 0) {
      f.state = 1;
      const int64_t st0 = f.start;
      stack.push_back({st0, n2, 0, {true, 0}, 0});
    } else if (f.state == 1) {
      f.state = 2;
      f.left = ret;
      f.hl = ret_h;
      const int64_t st1 = f.start + n2, n1 = f.n - n2;
      stack.push_back({st1, n1, 0, {true, 0}, 0});
    } else {
      const int32_t h = std::max(f.hl, ret_h) + 1;
      ints.push_back({f.left, ret, h});
      ret = {false, int32_t(ints.size() - 1)};
      ret_h = h;
      stack.pop_back();
    }
  }
  const int32_t L = int32_t(ls.size()), I = int32_t(ints.size());
  auto id_of = [&](const Ref& r) { return r.leaf ? r.idx : L + r.idx; };
  int32_t H = 0;
  for (const auto& in : ints) H = std::max(H, in.height);
  std::vector<int32_t> nid, nl, nr, off(size_t(H) + 1, 0);
  for (int32_t h = 1; h <= H; ++h) {
    off[size_t(h - 1)] = int32_t(nid.size());
    for (int32_t k = 0; k < I; ++k)
      if (ints[size_t(k)].height == h) {
        nid.push_back(L + k);
        nl.push_back(id_of(ints[size_t(k)].l));
        nr.push_back(id_of(ints[size_t(k)].r));
      }
  }
  off[size_t(H)] = int32_t(nid.size());
  auto* e = new ps_errsum;
  ps::ErrsumPlan& p = e->plan;
  p.rows_h = rows_h;
  p.cols_h = cols_h;
  p.count = N;
  p.nleaves = L;
  p.ninternal = I;
  p.nlevels = H;
  p.root = id_of(ret);
  p.h_level_off = off;
  bool ok = cudaMalloc(&p.leaf_start, sizeof(int64_t) * size_t(L)) == cudaSuccess &&
            cudaMalloc(&p.leaf_len, sizeof(int32_t) * size_t(L)) == cudaSuccess &&
            cudaMalloc(&p.node_left, sizeof(int32_t) * (size_t(I) + 1)) == cudaSuccess &&
            cudaMalloc(&p.node_right, sizeof(int32_t) * (size_t(I) + 1)) == cudaSuccess &&
            cudaMalloc(&p.node_id, sizeof(int32_t) * (size_t(I) + 1)) == cudaSuccess &&
            cudaMalloc(&p.level_off, sizeof(int32_t) * (size_t(H) + 1)) == cudaSuccess &&
            cudaMalloc(&p.values, sizeof(double) * 2 * size_t(L + I)) == cudaSuccess;
  ok = ok && cudaMemcpy(p.leaf_start, ls.data(), sizeof(int64_t) * size_t(L),
                        cudaMemcpyHostToDevice) == cudaSuccess;
  ok = ok && cudaMemcpy(p.leaf_len, ll.data(), sizeof(int32_t) * size_t(L),
                        cudaMemcpyHostToDevice) == cudaSuccess;
  if (I > 0) {
    ok = ok && cudaMemcpy(p.node_left, nl.data(), sizeof(int32_t) * size_t(I),
                          cudaMemcpyHostToDevice) == cudaSuccess;
    ok = ok && cudaMemcpy(p.node_right, nr.data(), sizeof(int32_t) * size_t(I),
                          cudaMemcpyHostToDevice) == cudaSuccess;
    ok = ok && cudaMemcpy(p.node_id, nid.data(), sizeof(int32_t) * size_t(I),
                          cudaMemcpyHostToDevice) == cudaSuccess;
  }
  ok = ok && cudaMemcpy(p.level_off, off.data(), sizeof(int32_t) * (size_t(H) + 1),
                        cudaMemcpyHostToDevice) == cudaSuccess;
  if (!ok) {
    ps_errsum_destroy(e);
    return nullptr;
  }
  return e;
}

void ps_errsum_destroy(ps_errsum* e) {
  if (!e) return;
  ps::ErrsumPlan& p = e->plan;
  cudaFree(p.leaf_start);
  cudaFree(p.leaf_len);
  cudaFree(p.node_left);
  cudaFree(p.node_right);
  cudaFree(p.node_id);
  cudaFree(p.level_off);
  cudaFree(p.values);
  delete e;
}

ps_status ps_errsum_step(ps_errsum* e, const ps_grid* g, const void* level, const void* S,
                         double st, double* out2, void* stream) {
  if (!e) return PS_ERR_ARG;
  ps_status s = check_grid(g);
  if (s != PS_OK) return s;
  if (!level || !S || !out2) return PS_ERR_ARG;
  if (g->dtype != PS_F64) return PS_ERR_ARG;
  const ps::ErrsumPlan& p = e->plan;
  const int64_t extra = g->bc == PS_BC_PERIODIC ? g->ghost : 0;
  if (p.rows_h > g->rows + extra || p.cols_h > g->cols + extra) return PS_ERR_SHAPE;
  cudaStream_t st_ = static_cast<cudaStream_t>(stream);
  const int32_t nvalues = p.nleaves + p.ninternal;
  k_errsum_leaves<<<unsigned((p.nleaves + 127) / 128), 128, 0, st_>>>(
      at_origin<double>(g, level), at_origin<double>(g, S), g->pitch, p.cols_h, st,
      p.leaf_start, p.leaf_len, p.nleaves, p.values, nvalues);
  k_errsum_fold<<<1, 1024, 0, st_>>>(p.node_left, p.node_right, p.node_id, p.level_off,
                                      p.nlevels, p.values, nvalues, p.root, out2);
  g_launches.fetch_add(2, std::memory_order_relaxed);
  return last_cuda_status();
}

ps_status ps_write_csv(const char* path, const void* host, int64_t rows, int64_t cols,
                       int64_t host_pitch, int32_t dtype) {
  // Host-side writer for dump_grid_csv (simulator.py:293-295: np.savetxt(fmt="%.17g",
  // delimiter=",")): one row per line, "%.17g" of each value widened to double.
  if (!path || !host || rows < 0 || cols < 0 || host_pitch < cols) return PS_ERR_ARG;
  if (dtype != PS_F64 && dtype != PS_F32) return PS_ERR_ARG;
  FILE* f = std::fopen(path, "w");
  if (!f) return PS_ERR_ARG;
  std::vector<char> line;
  line.reserve(size_t(cols) * 26 + 2);
  char buf[40];
  for (int64_t i = 0; i < rows; ++i) {
    line.clear();
    for (int64_t j = 0; j < cols; ++j) {
      const double x = dtype == PS_F64 ? static_cast<const double*>(host)[i * host_pitch + j]
                                       : double(static_cast<const float*>(host)[i * host_pitch + j]);
      const int len = std::snprintf(buf, sizeof(buf), "%.17g", x);
      if (j) line.push_back(',');
      line.insert(line.end(), buf, buf + len);
    }
    line.push_back('\n');
    if (std::fwrite(line.data(), 1, line.size(), f) != line.size()) {
      std::fclose(f);
      return PS_ERR_ARG;
    }
  }
  return std::fclose(f) == 0 ? PS_OK : PS_ERR_ARG;
}

int64_t ps_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

const char* ps_strerror(int32_t status) {
  switch (status) {
    case PS_OK: return "ok";
    case PS_ERR_ARG: return "invalid argument";
    case PS_ERR_SHAPE: return "grid shape does not fit the layout or the stencil";
    case PS_ERR_TABLE: return "coefficient table empty, too long, or wider than the ghost band";
    case PS_ERR_RADIUS: return "Dirichlet ring narrower than the stencil radius";
    case PS_ERR_CUDA: return "CUDA runtime error";
    case PS_ERR_ALIGN: return "level pointer not 16-byte aligned";
    default: return "unknown status";
  }
}

const char* ps_version(void) { return "paper_1904_04048_b200 0.1.0 sm_100a"; }

}  // extern "C"
