// ps_stream.cuh — stencil shapes and the streaming two-step kernel (the hot path).
// Included inside namespace ps by ps_device.cu.
//
// Persistent, warp-specialised row streaming: one producer warp issues TMA bulk copies
// (cp.async.bulk -> UBLKCP) of u^k row segments (+16-byte halo each side) and u^{k-1}
// row segments into an NS-stage shared-memory ring guarded by mbarrier transaction
// counts; NW consumer warps slide a (2R+1)-row register window down the strip, so every
// u^k element crosses HBM once and shared memory once; results leave as 16-byte stores;
// periodic edge points also write their wrap-around images.  Tap order and arithmetic
// follow the reference bit for bit (ps_arith.cuh); reference: simulator.py:147-205.
#pragma once

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

// Dynamic tile scheduler: one counter pair per in-flight launch.  The last block to
// finish resets its slot, so the next launch that reuses it starts from zero.  Slots are
// handed out by launch_slot() (ps_device.cu): direct launches cycle through
// [0, kDirectSlots) — safe while fewer than kDirectSlots launches of this library are in
// flight at once — and every kernel node of a captured CUDA graph owns a slot of
// [kDirectSlots, kSlots) that no direct launch or other graph uses (a graph's replays are
// serialised by CUDA, so its nodes never race with themselves).
constexpr int kSlots = 4096;
constexpr int kDirectSlots = 2048;
static __device__ unsigned int g_tile_next[kSlots];
static __device__ unsigned int g_tile_done[kSlots];

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

