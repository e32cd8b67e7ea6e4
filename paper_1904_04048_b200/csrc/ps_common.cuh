// ps_common.cuh — everything the kernel translation units share: the per-point
// contracts, the kernels (templates), host helpers, launchers and shape dispatch.
// ps_device.cu holds the C-ABI; ps_kern_{f64,f32r,f32n}.cu instantiate the streaming,
// temporal-blocking and first-step kernels for one (dtype, contract) each, so the three
// compile in parallel.
#pragma once
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

// launch accounting / per-launch tile-counter slots (defined in ps_device.cu)
extern std::atomic<int64_t> g_launches;
// Tile-counter slot of the next launch on `st` (ps_stream.cuh: g_tile_next/g_tile_done):
// direct launches cycle through [0, kDirectSlots); a launch recorded into a CUDA graph
// (stream capture) draws a slot from a separate pool that direct launches never touch and
// keeps it for the life of the graph.  -1: the graph pool is exhausted.
int launch_slot(cudaStream_t st);
// Device index clamped to the per-device caches below.
int device_index();

#include "ps_stream.cuh"

#include "ps_tblock.cuh"

#include "ps_generic.cuh"

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
constexpr int kMaxDevices = 64;
struct DevInfo {
  int nsm = 0;
};
inline DevInfo dev_info() {
  static std::mutex mu;
  static DevInfo cache[kMaxDevices];
  const int dev = device_index();
  std::lock_guard<std::mutex> lk(mu);
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

inline ps_status check_table(const ps_grid* g, const ps_table* t) {
  if (!t || t->ntaps < 1 || t->ntaps > PS_MAX_TAPS) return PS_ERR_TABLE;
  const int r = table_radius(t);
  if (r > g->ghost) return PS_ERR_TABLE;
  if (g->bc == PS_BC_DIRICHLET && r > g->ring) return PS_ERR_RADIUS;
  return PS_OK;
}

inline ps_status check_grid(const ps_grid* g) {
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
// Peer halo targets of a temporally blocked row-slab pass (allocation bases of the
// neighbours' out_prev / out_last levels, as from ps_ipc_open; null = none).
struct TBHalo {
  void* up_prev = nullptr;
  void* up_last = nullptr;
  void* dn_prev = nullptr;
  void* dn_last = nullptr;
  int32_t up_rows = 0;
};

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
  // the shared-memory opt-in is a per-device function attribute: once per device
  static std::once_flag once[kMaxDevices];
  static int bps[kMaxDevices];
  const int dev = device_index();
  std::call_once(once[dev], [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Gm::smem_bytes));
    bps[dev] = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps[dev], kern, (NW + 1) * 32,
                                                  Gm::smem_bytes);
    if (bps[dev] < 1) bps[dev] = 1;
  });
  const int blocks_per_sm = bps[dev];
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
  const int slot = launch_slot(st);
  if (slot < 0) return PS_ERR_CUDA;
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

// ---------------------------------------------------------------------------
// Temporal blocking (ps_tblock.cuh)
// ---------------------------------------------------------------------------
// Geometry (measured on B200, tools/tb_variants.sh): 11 consumer warps + 1
// producer warp, one block per SM, 3 pipeline stages.  Tuning builds override with -D.
#ifndef PS_TB_NW
#define PS_TB_NW 0
#endif
#ifndef PS_TUNE_BC
#define PS_TUNE_BC PS_BC_DIRICHLET
#endif
#ifndef PS_TB_RC_ALIGN
#define PS_TB_RC_ALIGN 1  // 0: keep the round tile heights
#endif
#ifndef PS_TB_RB
#define PS_TB_RB 0  // 0: per radius (launch_tb)
#endif
#ifndef PS_TB_NS
#define PS_TB_NS 0
#endif
#ifndef PS_TB_VM
#define PS_TB_VM 0
#endif
// 16-byte vectors per lane (TBGeom VM).  Measured (C4, f64 P9 T=4, 40 steps): two vectors
// per lane in 7 consumer warps (8 warps per SM -> up to 255 registers, no spills) 585 vs
// 535 GLUP/s for one vector in 11 warps (168 registers); P13 f64 (358 vs 368), f32 (708
// vs 1008: spills) and periodic grids (C2: 251 vs 324) stay at one vector.  Folding the
// producer into consumer warp 0 (8 consumer warps, 2 per sub-partition) lost everywhere
// (C4 528, C5 801).
#ifndef PS_TB_SYM_VM
#define PS_TB_SYM_VM 1   // vectors per lane of the shared-product kernels (state: 15 doubles
#endif                   // per stage at one f64 vector, 27 at two: T=4 fits only with one)
#ifndef PS_TB_SYM_WGS
#define PS_TB_SYM_WGS 1  // shared-product kernels: 12 warpgroup-specialised consumer warps
#endif
template <typename T, int A, class S, int TS, bool PER>
constexpr int tb_vm() {
  return PS_TB_VM > 0            ? PS_TB_VM
         : tb_sym<T, A, S, TS, PER>()     ? PS_TB_SYM_VM
                                 : ((sizeof(T) == 8 && S::R == 1 && !PER) ? 2 : 1);
}
#ifndef PS_TB_WGS
#define PS_TB_WGS -1
#endif
// warpgroup-specialised block (k_two_step_tb WGS).  Measured (40 steps): C4 616-625 vs
// 579-600 GLUP/s for 7 consumers + a producer warp (200-step bench: 593 vs 564); f32 with
// 12 consumers (160 registers): C5 1036 -> 1052, C3 f32 804 -> 826; P13 f64 unchanged
// (370-376), periodic C2 slower (321 -> 291), so those keep 11 consumers + a producer.
#ifndef PS_TB_WGS1
#define PS_TB_WGS1 -1  // one-vector geometries: 1 = always, 0 = never, -1 = f32 Dirichlet
#endif
// f64 radius-2 passes of depth >= 3 keep 3-4 five-row windows (90-120 doubles): they fit
// the 232 registers of 8 warpgroup-specialised consumer warps without spilling (C3 T=3 381,
// T=4 360 GLUP/s; 11 warps x 168 registers spilled 456 B at T=4: 319)
template <typename T, class S, int TS>
constexpr bool tb_deep_r2() {
  return sizeof(T) == 8 && S::R == 2 && TS >= 3;
}
template <typename T, int A, class S, int TS, bool PER>
constexpr bool tb_wgs() {
  return PS_TB_WGS >= 0 ? PS_TB_WGS != 0
         : tb_vm<T, A, S, TS, PER>() == 2
             ? true
             : (tb_sym<T, A, S, TS, PER>() ? (PS_TB_SYM_WGS == 2 || (PS_TB_SYM_WGS != 0 && !PER))
                : (PS_TB_WGS1 >= 0 ? PS_TB_WGS1 != 0
                                   : ((sizeof(T) == 4 || tb_deep_r2<T, S, TS>()) && !PER)));
}
#ifndef PS_TB_WGS_NW
#define PS_TB_WGS_NW 0   // tuning: consumer warps of a warpgroup-specialised block (8 or 12)
#endif
template <typename T, int A, class S, int TS, bool PER>
constexpr int tb_nw() {
  // shared-product kernels: 8 consumer warps x 232 registers (no spills; 12 x 160 spill
  // 80-116 B: C4 600 vs 568 GLUP/s on the 200-step run)
  return tb_wgs<T, A, S, TS, PER>() ? (PS_TB_WGS_NW > 0 ? PS_TB_WGS_NW
                                       : (tb_vm<T, A, S, TS, PER>() == 2 ||
                                          tb_deep_r2<T, S, TS>() || tb_sym<T, A, S, TS, PER>())
                                           ? 8 : 12)
         : PS_TB_NW > 0             ? PS_TB_NW
                                    : (tb_vm<T, A, S, TS, PER>() == 2 ? 7 : 11);
}
template <typename T, int TS, bool SYM = false>
constexpr int tb_ns() {
  return PS_TB_NS > 0 ? PS_TB_NS : 3;
}

template <typename T, int A, class S, int TS, bool PER, bool HALO>
static ps_status launch_tb(const ps_grid* g, const void* uk, const void* ukm1, void* out_prev,
                           void* out_last, const ps_table* t, int64_t rlo, int64_t rhi,
                           cudaStream_t st, bool reverse, int rc_hint, const TBHalo& h) {
  constexpr bool SYM = tb_sym<T, A, S, TS, PER>();
  constexpr int VM = tb_vm<T, A, S, TS, PER>(), NW = tb_nw<T, A, S, TS, PER>();
  constexpr int NS = tb_ns<T, TS, SYM>();
  constexpr bool WGS = tb_wgs<T, A, S, TS, PER>();
  if (SYM && !tb_classes_equal<S>(t)) return PS_ERR_TABLE;  // (tb_supported screens these)
  constexpr int NT = (NW + (WGS ? 4 : 1)) * 32;  // threads per block (consumers + producer)
  // rows per pipeline slot: one window rotation (2R+1) for radius 1; radius 2 takes 6
  // (measured: C5 1052 -> 1080, C3 f32 827 -> 837 GLUP/s; fewer ring waits per row, and
  // 8 or 10 rows no longer fit the shared memory)
  // shared-product kernels rotate 2R-row delay lines: a multiple of 2R rows per slot
  // (8 warps: 8 rows x 3 slots 664-692 GLUP/s on C4, 8 x 2 573-583, 4 x 3 603-606)
  // radius 1: 10 rows x 3 slots where they fit the 227 KB (depths >= 4: narrower strips) --
  // C4 T=5 772 vs 756 GLUP/s at full clocks (6 x 4: 737, 4 x 6: 718: the per-slot
  // wait/arrive round is what costs, so fewer, taller slots)
  constexpr int RBS =
      (S::R == 1 && TBGeom<T, NW, 10, NS, S::R, TS, VM>::smem_bytes <= size_t(227) * 1024) ? 10 : 8;
  constexpr int RB = PS_TB_RB > 0 ? PS_TB_RB : SYM ? RBS : (S::R == 2 ? 6 : 2 * S::R + 1);
  using Gm = TBGeom<T, NW, RB, NS, S::R, TS, VM>;
  auto kern = k_two_step_tb<T, A, S, TS, PER, HALO, NW, RB, NS, VM, WGS>;
  static std::once_flag once[kMaxDevices];
  static int bps[kMaxDevices];
  const int dev = device_index();
  std::call_once(once[dev], [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Gm::smem_bytes));
    bps[dev] = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps[dev], kern, NT, Gm::smem_bytes);
    if (bps[dev] < 1) bps[dev] = 1;
  });
  const int blocks_per_sm = bps[dev];
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
  p.row_images = (PER && single_slab(g)) ? 1 : 0;
  p.hu_prev = h.up_prev ? at_origin<T>(g, h.up_prev) : nullptr;
  p.hu_last = h.up_last ? at_origin<T>(g, h.up_last) : nullptr;
  p.hd_prev = h.dn_prev ? at_origin<T>(g, h.dn_prev) : nullptr;
  p.hd_last = h.dn_last ? at_origin<T>(g, h.dn_last) : nullptr;
  p.up_rows = h.up_rows;
  for (int s = 0; s < S::N; ++s) {
    p.c[s] = t->c[s];
    p.cf[s] = static_cast<float>(t->c[s]);
  }
  const int resident = std::max(1, dev_info().nsm) * blocks_per_sm;
  p.nstrips = int32_t((g->cols + Gm::W - 1) / Gm::W);
  int rc = env_int("PS_TB_ROW_CHUNK", 0);
  if (rc <= 0) rc = rc_hint;  // banded solve (ps_solve.cuh): its own tile height
  const bool rc_auto = rc <= 0;
  if (rc_auto) {
    const int64_t want_tiles = int64_t(resident) * 8;
    const int64_t chunks = (want_tiles + p.nstrips - 1) / p.nstrips;
    rc = int(std::max<int64_t>(1, (nrows + chunks - 1) / chunks));
    rc = std::max(rc, std::max(32, 8 * S::R * TS));
    rc = std::min(rc, 256);
    // very tall grids: taller tiles recompute fewer halo rows per pass (C5: +3 %), as
    // long as every block still gets >= 32 tiles for the dynamic balance
    for (const int tall : {512, 384})
      if (rc == 256 && int64_t(p.nstrips) * ((nrows + tall - 1) / tall) >= 32 * int64_t(resident)) {
        rc = tall;
        break;
      }
  }
  // a tile streams rc + 2*R*TS rows: make that a whole number of pipeline slots, so the
  // tile's last slot is a full (unrolled) one
  if (PS_TB_RC_ALIGN && rc_auto && rc >= 8 * RB)
    rc += (RB - (rc + 2 * S::R * TS) % RB) % RB;
  rc = int(std::min<int64_t>(rc, nrows));
  p.rc = rc;
  p.ntiles = int32_t(((nrows + rc - 1) / rc) * p.nstrips);
  const int grid = int(std::min<int64_t>(p.ntiles, resident));
  const int slot = launch_slot(st);
  if (slot < 0) return PS_ERR_CUDA;
  if (launch_pdl(kern, grid, NT, Gm::smem_bytes, st, p, slot) != cudaSuccess)
    return PS_ERR_CUDA;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return last_cuda_status();
}

template <typename T, int A, int TS, class S>
static ps_status launch_tb_bc(const ps_grid* g, const void* uk, const void* ukm1, void* op,
                              void* ol, const ps_table* t, int64_t lo, int64_t hi,
                              cudaStream_t st, bool rev, int rc, const TBHalo& h) {
  if (g->bc == PS_BC_PERIODIC)
    return launch_tb<T, A, S, TS, true, false>(g, uk, ukm1, op, ol, t, lo, hi, st, rev, rc, h);
  if (h.up_prev || h.up_last || h.dn_prev || h.dn_last)
    return launch_tb<T, A, S, TS, false, true>(g, uk, ukm1, op, ol, t, lo, hi, st, rev, rc, h);
  return launch_tb<T, A, S, TS, false, false>(g, uk, ukm1, op, ol, t, lo, hi, st, rev, rc, h);
}

template <typename T, int A, int TS>
static ps_status dispatch_tb(const ps_grid* g, const void* uk, const void* ukm1, void* op,
                             void* ol, const ps_table* t, int64_t lo, int64_t hi,
                             cudaStream_t st, bool rev, int rc, const TBHalo& h) {
#ifdef PS_TUNE_SHAPE
  // tuning builds (tools/tb_variants.sh) instantiate ONE fused kernel: the plain pass of
  // PS_TUNE_SHAPE at depth PS_TUNE_TS; everything else reports "unsupported"
  if constexpr (TS == PS_TUNE_TS) {
    if (shape_matches<PS_TUNE_SHAPE>(t) && g->bc == PS_TUNE_BC)
      return launch_tb<T, A, PS_TUNE_SHAPE, TS, PS_TUNE_BC == PS_BC_PERIODIC, false>(
          g, uk, ukm1, op, ol, t, lo, hi, st, rev, rc, h);
  }
  return PS_ERR_TABLE;
#else
  if constexpr (TS >= 5) {
    // deep fusion: shared-product kernels only (their 15-double stage state is what makes
    // five or six stages fit 232 registers), Dirichlet, plain pass or in-kernel halo pass
    if (g->bc != PS_BC_DIRICHLET) return PS_ERR_ARG;
    const bool halo = h.up_prev || h.up_last || h.dn_prev || h.dn_last;
    auto go = [&](auto shape) -> ps_status {
      using S = decltype(shape);
      if constexpr (tb_sym<T, A, S, TS, false>()) {
        if (halo)
          return launch_tb<T, A, S, TS, false, true>(g, uk, ukm1, op, ol, t, lo, hi, st, rev, rc, h);
        return launch_tb<T, A, S, TS, false, false>(g, uk, ukm1, op, ol, t, lo, hi, st, rev, rc, h);
      } else {
        return PS_ERR_ARG;
      }
    };
    if (shape_matches<ShapeP5>(t)) return go(ShapeP5{});
    if (shape_matches<ShapeP9>(t)) return go(ShapeP9{});
    if (shape_matches<ShapeC9>(t)) return go(ShapeC9{});
    return PS_ERR_TABLE;
  } else {  // (an else branch, so depths 5 and 6 do not instantiate the kernels below)
    if (shape_matches<ShapeP5>(t))
      return launch_tb_bc<T, A, TS, ShapeP5>(g, uk, ukm1, op, ol, t, lo, hi, st, rev, rc, h);
    if (shape_matches<ShapeP9>(t))
      return launch_tb_bc<T, A, TS, ShapeP9>(g, uk, ukm1, op, ol, t, lo, hi, st, rev, rc, h);
    if (shape_matches<ShapeC9>(t))
      return launch_tb_bc<T, A, TS, ShapeC9>(g, uk, ukm1, op, ol, t, lo, hi, st, rev, rc, h);
    if (shape_matches<ShapeP13>(t))
      return launch_tb_bc<T, A, TS, ShapeP13>(g, uk, ukm1, op, ol, t, lo, hi, st, rev, rc, h);
    return PS_ERR_TABLE;
  }
#endif
}

// First step as two streaming launches: u1 <- -fl(tau * A_v(v0)) (VP), then the ordinary
// two-step kernel u1 <- fl(A_u(u0) - u1) = fl(A_u(u0) + fl(tau * A_v(v0))), bit for bit the
// reference's first step.  Both tables must have a specialised shape.
template <typename T, int A, bool PER>
static ps_status first_step_stream(const ps_grid* g, const void* u0, const void* v0, void* u1,
                                   const ps_table* tu, const ps_table* tv, double tau,
                                   int64_t lo, int64_t hi, cudaStream_t st, bool* done) {
  *done = true;
  const Halo h;
  ps_status s;
  if (shape_matches<ShapeP5>(tv))
    s = launch_stream<T, A, ShapeP5, PER, true>(g, v0, v0, u1, tv, lo, hi, st, h, tau);
  else if (shape_matches<ShapeP9>(tv))
    s = launch_stream<T, A, ShapeP9, PER, true>(g, v0, v0, u1, tv, lo, hi, st, h, tau);
  else if (shape_matches<ShapeC9>(tv))
    s = launch_stream<T, A, ShapeC9, PER, true>(g, v0, v0, u1, tv, lo, hi, st, h, tau);
  else if (shape_matches<ShapeP13>(tv))
    s = launch_stream<T, A, ShapeP13, PER, true>(g, v0, v0, u1, tv, lo, hi, st, h, tau);
  else {
    *done = false;
    return PS_OK;
  }
  if (s != PS_OK) return s;
  return dispatch_two_step<T, A, PER>(g, u0, u1, u1, tu, lo, hi, st, h);
}


// ---------------------------------------------------------------------------
// Typed entry points, one translation unit per (dtype, contract): ps_kern_*.cu
// ---------------------------------------------------------------------------
// One translation unit per (dtype, contract) for the streaming / first-step kernels, and
// one per (dtype, contract, depth) for the fused kernels (ps_kern_*_t<depth>.cu): twelve
// units that compile in parallel instead of three long ones.
#define PS_TYPED_DECL(SFX)                                                                  \
  ps_status two_step_##SFX(const ps_grid* g, const void* uk, const void* ukm1, void* ukp1,  \
                           const ps_table* t, int64_t lo, int64_t hi, cudaStream_t st,      \
                           const Halo& h);                                                  \
  ps_status tb_##SFX##_t2(const ps_grid* g, const void* uk, const void* ukm1, void* op,     \
                          void* ol, const ps_table* t, int64_t lo, int64_t hi,              \
                          cudaStream_t st, bool rev, int rc, const TBHalo& h);              \
  ps_status tb_##SFX##_t3(const ps_grid* g, const void* uk, const void* ukm1, void* op,     \
                          void* ol, const ps_table* t, int64_t lo, int64_t hi,              \
                          cudaStream_t st, bool rev, int rc, const TBHalo& h);              \
  ps_status tb_##SFX##_t4(const ps_grid* g, const void* uk, const void* ukm1, void* op,     \
                          void* ol, const ps_table* t, int64_t lo, int64_t hi,              \
                          cudaStream_t st, bool rev, int rc, const TBHalo& h);              \
  ps_status tb_##SFX##_t5(const ps_grid* g, const void* uk, const void* ukm1, void* op,     \
                          void* ol, const ps_table* t, int64_t lo, int64_t hi,              \
                          cudaStream_t st, bool rev, int rc, const TBHalo& h);              \
  ps_status tb_##SFX##_t6(const ps_grid* g, const void* uk, const void* ukm1, void* op,     \
                          void* ol, const ps_table* t, int64_t lo, int64_t hi,              \
                          cudaStream_t st, bool rev, int rc, const TBHalo& h);              \
  inline ps_status tb_##SFX(const ps_grid* g, const void* uk, const void* ukm1, void* op,   \
                            void* ol, const ps_table* t, int tsteps, int64_t lo, int64_t hi, \
                            cudaStream_t st, bool rev, int rc, const TBHalo& h) {           \
    switch (tsteps) {                                                                       \
      case 2: return tb_##SFX##_t2(g, uk, ukm1, op, ol, t, lo, hi, st, rev, rc, h);         \
      case 3: return tb_##SFX##_t3(g, uk, ukm1, op, ol, t, lo, hi, st, rev, rc, h);         \
      case 4: return tb_##SFX##_t4(g, uk, ukm1, op, ol, t, lo, hi, st, rev, rc, h);         \
      case 5: return tb_##SFX##_t5(g, uk, ukm1, op, ol, t, lo, hi, st, rev, rc, h);         \
      case 6: return tb_##SFX##_t6(g, uk, ukm1, op, ol, t, lo, hi, st, rev, rc, h);         \
      default: return PS_ERR_ARG;                                                           \
    }                                                                                       \
  }                                                                                         \
  ps_status first_##SFX(const ps_grid* g, const void* u0, const void* v0, void* u1,         \
                        const ps_table* tu, const ps_table* tv, double tau, int64_t lo,     \
                        int64_t hi, cudaStream_t st, bool* done);
PS_TYPED_DECL(f64)
PS_TYPED_DECL(f32r)
PS_TYPED_DECL(f32n)
#undef PS_TYPED_DECL

#define PS_TYPED_DEFINE(SFX, T, A)                                                          \
  ps_status two_step_##SFX(const ps_grid* g, const void* uk, const void* ukm1, void* ukp1,  \
                           const ps_table* t, int64_t lo, int64_t hi, cudaStream_t st,      \
                           const Halo& h) {                                                 \
    return dispatch_two_step_bc<T, A>(g, uk, ukm1, ukp1, t, lo, hi, st, h);                 \
  }                                                                                         \
  ps_status first_##SFX(const ps_grid* g, const void* u0, const void* v0, void* u1,         \
                        const ps_table* tu, const ps_table* tv, double tau, int64_t lo,     \
                        int64_t hi, cudaStream_t st, bool* done) {                          \
    return g->bc == PS_BC_PERIODIC                                                          \
               ? first_step_stream<T, A, true>(g, u0, v0, u1, tu, tv, tau, lo, hi, st, done) \
               : first_step_stream<T, A, false>(g, u0, v0, u1, tu, tv, tau, lo, hi, st, done); \
  }

// depths 5 and 6 exist for the shared-product kernels only (f64, radius 1, Dirichlet);
// the other contracts define stubs
#define PS_TYPED_DEFINE_TB_STUB(SFX, TS)                                                    \
  ps_status tb_##SFX##_t##TS(const ps_grid*, const void*, const void*, void*, void*,        \
                             const ps_table*, int64_t, int64_t, cudaStream_t, bool, int,    \
                             const TBHalo&) {                                               \
    return PS_ERR_ARG;                                                                      \
  }

#define PS_TYPED_DEFINE_TB(SFX, T, A, TS)                                                   \
  ps_status tb_##SFX##_t##TS(const ps_grid* g, const void* uk, const void* ukm1, void* op,  \
                             void* ol, const ps_table* t, int64_t lo, int64_t hi,           \
                             cudaStream_t st, bool rev, int rc, const TBHalo& h) {          \
    return dispatch_tb<T, A, TS>(g, uk, ukm1, op, ol, t, lo, hi, st, rev, rc, h);           \
  }

}  // namespace ps
