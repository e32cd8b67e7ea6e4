// ps_tile.cuh — tile-resident march for small f64 grids, Dirichlet or periodic (BASELINE config 1: the
// reference's own regime, n <= a few hundred).  Included inside namespace ps by ps_device.cu.
//
// A 512^2 level is 2 MB: it lives in L2, and one streaming launch per step costs a launch
// round trip (4.1 us with CUDA-graph replay + PDL) for 0.2 us of arithmetic.  Here the grid
// is cut into py x px tiles, one CTA (= one SM) per tile, all co-resident (cooperative
// launch).  A pass ("epoch") of T updates:
//   1. wait until the 8 neighbouring tiles have published the previous epoch,
//   2. load the tile plus a halo of H = R*T points of u^k and u^{k-1} into shared memory
//      (ld.global.cg: the neighbours' rows come from L2, never from a stale L1 line),
//   3. run T updates in shared memory on regions shrinking by R per update (the halo
//      points are recomputed redundantly, like the fused streaming kernel's columns),
//   4. store the tile of u^{k+T-1} and u^{k+T} to the OTHER pair of levels, fence, and
//      publish the epoch number.
// Epoch e reads pair e&1 and writes pair (e+1)&1, so a tile never overwrites rows a
// neighbour may still be loading: a neighbour starts epoch e+1 (which writes the pair this
// tile reads in epoch e) only after this tile published e+1, i.e. finished epoch e.
// The per-point arithmetic is Arith<double, REF>::tap over the compile-time tap list of the
// scheme shape with run-time coefficients — the same sequence as every other kernel, so the
// result equals T single launches bit for bit; the Dirichlet ring is re-pinned to +0.0 at
// every update (simulator.py:147-160, 183-191).  Periodic grids: tiles form a ring in both
// directions, halos are loaded with wrapped indices from the n x n core, and ps_march_tile
// refreshes the wrap-around images of the two final levels afterwards (ps_fill_ghosts).
//
// Measured on the B200 (C1: P5, 512^2, 200 steps, 13 x 11 tiles of 40 x 47): 1.94 us per step
// at T = 10..12 (134 GLUP/s) against 4.06-4.4 for the CUDA-graph-replayed streaming march;
// of the 2.2 us at T = 8, 0.95 is the updates (shared-memory bandwidth: a (2R+1)^2 register
// window per thread cut P5's loads per point from 6 to 4), 0.53 the neighbour wait, 0.38
// the global loads/stores and 0.5 launch + fences.

struct TileParams {
  void* lvl[4];           // logical (0,0) of the four levels
  int64_t pitch;
  int32_t rows, cols, ring;
  int32_t py, px, th, tw;  // tiles and their nominal height/width (last ones shorter)
  int32_t nepochs, T, last_T;
  int32_t in_cur, in_prev, out_cur, out_prev;  // epoch 0 reads (in_*), writes (out_*)
  unsigned int* flags;    // [py*px], zero on entry
  double c[PS_MAX_TAPS];
};

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

constexpr int kTileThreads = 512;
constexpr int kTileLanes = 64;  // threads along a row

template <class S, bool PER>
__global__ void __launch_bounds__(kTileThreads, 1) k_tile_march(const __grid_constant__ TileParams p) {
  constexpr int R = S::R;
  using Ar = Arith<double, ARITH_REF>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int H = R * p.T;
  const int SH = p.th + 2 * H, SP = p.tw + 2 * H;  // shared-memory tile: rows x pitch
  double* const base = reinterpret_cast<double*>(smem_raw);
  const int BS = SH * SP;  // elements per shared-memory level

  const int ty0 = blockIdx.x / p.px, tx0 = blockIdx.x - ty0 * p.px;
  const int r0 = ty0 * p.th, r1 = min(r0 + p.th, p.rows);
  const int c0 = tx0 * p.tw, c1 = min(c0 + p.tw, p.cols);
  const int tid = threadIdx.x;
  const int ty = tid / kTileLanes, tx = tid - ty * kTileLanes;
  constexpr int NY = kTileThreads / kTileLanes;

  double c[S::N];
#pragma unroll
  for (int s = 0; s < S::N; ++s) c[s] = p.c[s];

  // the (up to) 8 neighbouring tiles whose epochs this tile waits for
  int nb = -1;
  if (tid < 9 && tid != 4) {
    int ny = ty0 + tid / 3 - 1, nx = tx0 + tid % 3 - 1;
    if (PER) {  // a ring of tiles in both directions (a tile may be its own neighbour)
      ny = (ny + p.py) % p.py;
      nx = (nx + p.px) % p.px;
    }
    if (ny >= 0 && ny < p.py && nx >= 0 && nx < p.px) nb = ny * p.px + nx;
  }

  int in_cur = p.in_cur, in_prev = p.in_prev, out_cur = p.out_cur, out_prev = p.out_prev;
  for (int e = 0; e < p.nepochs; ++e) {
    const int Te = (e == p.nepochs - 1) ? p.last_T : p.T;
    if (e > 0) {
      if (nb >= 0)
        while (ld_acquire_u32(p.flags + nb) < unsigned(e)) {
        }
      __syncthreads();
    }
    // ---- load u^k -> level 1, u^{k-1} -> level 0 on the tile + R*Te halo (0 outside the grid)
    {
      const int E = R * Te;
      const double* gk = static_cast<const double*>(p.lvl[in_cur]);
      const double* gm = static_cast<const double*>(p.lvl[in_prev]);
      const int i_lo = r0 - E, i_hi = r1 + E, j_lo = c0 - E, j_hi = c1 + E;
      // four rows per thread in flight: the L2 round trips overlap instead of queueing
      constexpr int U = 4;
      for (int i = i_lo + ty; i < i_hi; i += U * NY) {
        for (int j = j_lo + tx; j < j_hi; j += kTileLanes) {
          const int lj = j - (c0 - H);
          double a[U], b[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int ii = i + u * NY;
            a[u] = b[u] = 0.0;
            if (PER) {
              if (ii < i_hi) {   // periodic: the halo wraps around the core (no images read)
                const int iw = ii < 0 ? ii + p.rows : (ii >= p.rows ? ii - p.rows : ii);
                const int jw = j < 0 ? j + p.cols : (j >= p.cols ? j - p.cols : j);
                a[u] = __ldcg(gk + int64_t(iw) * p.pitch + jw);
                b[u] = __ldcg(gm + int64_t(iw) * p.pitch + jw);
              }
            } else if (ii < i_hi && ii >= 0 && ii < p.rows && j >= 0 && j < p.cols) {
              a[u] = __ldcg(gk + int64_t(ii) * p.pitch + j);
              b[u] = __ldcg(gm + int64_t(ii) * p.pitch + j);
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int ii = i + u * NY;
            if (ii < i_hi) {
              const int li = ii - (r0 - H);
              base[BS + li * SP + lj] = a[u];
              base[li * SP + lj] = b[u];
            }
          }
        }
      }
    }
    __syncthreads();
    // ---- Te updates in shared memory
    int cur = 1, prev = 0, nxt = 2;
    for (int s = 1; s <= Te; ++s) {
      const int E = R * (Te - s);
      const int i_lo = PER ? r0 - E : max(r0 - E, 0), i_hi = PER ? r1 + E : min(r1 + E, p.rows);
      const int j_lo = PER ? c0 - E : max(c0 - E, 0), j_hi = PER ? c1 + E : min(c1 + E, p.cols);
      const double* __restrict__ L = base + cur * BS;
      const double* __restrict__ M = base + prev * BS;
      double* __restrict__ O = base + nxt * BS;
      // Each thread walks a band of consecutive rows of one column with a (2R+1)^2 register
      // window: a new row costs 2R+1 shared-memory loads (+1 for u^{k-1}) instead of one per
      // tap -- the update is shared-memory-bandwidth bound (P5: 6 -> 4 loads per point).
      // Sums are computed unconditionally (a ring point's taps stay inside the
      // shared-memory level: E <= H - R) and masked afterwards.
      constexpr int WN = 2 * R + 1;
      const int bh = (i_hi - i_lo + NY - 1) / NY;
      const int b0 = i_lo + ty * bh, b1 = min(b0 + bh, i_hi);
      for (int j = j_lo + tx; j < j_hi; j += kTileLanes) {
        const int lj = j - (c0 - H);
        const bool col_in = PER || (j >= p.ring && j < p.cols - p.ring);
        double win[WN][WN];
#pragma unroll
        for (int r = 0; r + 1 < WN; ++r)
#pragma unroll
          for (int x = 0; x < WN; ++x)
            win[r + 1][x] = (b0 < b1) ? L[(b0 - (r0 - H) - R + r) * SP + lj - R + x] : 0.0;
        // WN rows per trip with the window rotating through compile-time slots (logical row
        // r of trip step u lives in slot (r + 1 + u) % WN), so no register moves
        for (int ib = b0; ib < b1; ib += WN) {
#pragma unroll
          for (int u = 0; u < WN; ++u) {
            const int i = ib + u;
            if (i < b1) {
              const int li = i - (r0 - H);
#pragma unroll
              for (int x = 0; x < WN; ++x) win[u % WN][x] = L[(li + R) * SP + lj - R + x];
              double acc = Ar::zero();
#pragma unroll
              for (int q = 0; q < S::N; ++q)
                acc = Ar::tap(acc, c[q], win[(R + S::q(q, 0) + 1 + u) % WN][R + S::q(q, 1)]);
              const double r = Ar::two(acc, M[li * SP + lj]);
              O[li * SP + lj] = (col_in && (PER || (i >= p.ring && i < p.rows - p.ring))) ? r : 0.0;
            }
          }
        }
      }
      __syncthreads();
      const int t = prev;
      prev = cur;
      cur = nxt;
      nxt = t;
    }
    // ---- store the tile of the two newest levels to the other pair and publish
    {
      double* gc = static_cast<double*>(p.lvl[out_cur]);
      double* gp = static_cast<double*>(p.lvl[out_prev]);
      for (int i = r0 + ty; i < r1; i += NY) {
        const int li = i - (r0 - H);
        for (int j = c0 + tx; j < c1; j += kTileLanes) {
          const int lj = j - (c0 - H);
          gc[int64_t(i) * p.pitch + j] = base[cur * BS + li * SP + lj];
          gp[int64_t(i) * p.pitch + j] = base[prev * BS + li * SP + lj];
        }
      }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release_u32(p.flags + blockIdx.x, unsigned(e + 1));
    int t = in_cur;
    in_cur = out_cur;
    out_cur = t;
    t = in_prev;
    in_prev = out_prev;
    out_prev = t;
  }
}

// Tiling for a rows x cols grid at depth T on nsm SMs: py x px <= nsm tiles, each at least
// R*T tall and wide (a halo reaches only the adjacent tiles), three (th+2H) x (tw+2H) f64
// buffers within max_smem; among those the least work per update.  false = no fit.
static bool tile_plan(int64_t rows, int64_t cols, int R, int T, int nsm, size_t max_smem,
                      int* py, int* px, int* th, int* tw, size_t* smem) {
  const int H = R * T;
  double best = 0;
  bool ok = false;
  for (int y = 1; y <= nsm; ++y) {
    const int x = nsm / y;
    if (x < 1) break;
    const int h = int((rows + y - 1) / y), w = int((cols + x - 1) / x);
    if (h < H || w < H) continue;
    // (the last tile row/column may be shorter than H only if it is empty)
    const int64_t last_h = rows - int64_t(h) * ((rows + h - 1) / h - 1);
    const int64_t last_w = cols - int64_t(w) * ((cols + w - 1) / w - 1);
    if (last_h < H || last_w < H) continue;
    const size_t bytes = size_t(3) * (h + 2 * H) * (w + 2 * H) * sizeof(double);
    if (bytes > max_smem) continue;
    // cost: rows of the halo region x 64-lane column chunks
    const double cost = double(h + 2 * H) * double((w + 2 * H + kTileLanes - 1) / kTileLanes);
    if (!ok || cost < best) {
      ok = true;
      best = cost;
      *py = int((rows + h - 1) / h);
      *px = int((cols + w - 1) / w);
      *th = h;
      *tw = w;
      *smem = bytes;
    }
  }
  return ok;
}

template <class S, bool PER>
static ps_status launch_tile(const ps_grid* g, void* lvl[4], int64_t nsteps, const ps_table* t,
                             int T, int cur, int prev, int f_prev, int f_cur, unsigned int* flags,
                             cudaStream_t st, int py, int px, int th, int tw, size_t smem) {
  auto kern = k_tile_march<S, PER>;
  static std::once_flag once[kMaxDevices];
  const int dev = device_index();
  std::call_once(once[dev], [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  });
  TileParams p;
  std::memset(&p, 0, sizeof(p));
  for (int x = 0; x < 4; ++x) p.lvl[x] = at_origin<double>(g, lvl[x]);
  p.pitch = g->pitch;
  p.rows = int32_t(g->rows);
  p.cols = int32_t(g->cols);
  p.ring = g->ring;
  p.py = py;
  p.px = px;
  p.th = th;
  p.tw = tw;
  p.T = T;
  p.nepochs = int32_t((nsteps + T - 1) / T);
  p.last_T = int32_t(nsteps - int64_t(p.nepochs - 1) * T);
  p.in_cur = cur;
  p.in_prev = prev;
  p.out_cur = f_cur;
  p.out_prev = f_prev;
  p.flags = flags;
  for (int s = 0; s < S::N; ++s) p.c[s] = t->c[s];
  if (cudaMemsetAsync(flags, 0, sizeof(unsigned int) * size_t(py) * px, st) != cudaSuccess)
    return PS_ERR_CUDA;
  void* args[] = {&p};
  if (cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(unsigned(py * px)),
                                  dim3(kTileThreads), args, smem, st) != cudaSuccess)
    return PS_ERR_CUDA;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return last_cuda_status();
}
