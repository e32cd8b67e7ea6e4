// ps_device.cu — host side of libps.so: launch configuration, dispatch by stencil shape,
// CUDA-graph replay, and the C-ABI declared in include/ps.h.  The kernels live in
//   ps_stream.cuh   streaming two-step kernel (the hot path; also the first step's halves)
//   ps_tblock.cuh   temporal blocking (T fused updates per pass)
//   ps_generic.cuh  runtime-table kernel, periodic image refresh, Gaussian initial data
//   ps_errsum.cuh   run()'s per-step error sums in numpy's pairwise order
//   ps_solve.cuh    host-to-host solve: banded wavefront with the PCIe copies overlapped
// with ps_arith.cuh (the per-point arithmetic contracts) and ps_ptx.cuh (mbarrier, TMA,
// PDL primitives).
#include "ps_common.cuh"

namespace ps {

std::atomic<int64_t> g_launches{0};

int device_index() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) cudaGetLastError();
  return (dev < 0 || dev >= kMaxDevices) ? 0 : dev;
}

// Tile-counter slots (ps_stream.cuh).  Direct launches: a sequence number modulo
// kDirectSlots.  Launches recorded by stream capture: a slot of the graph pool, returned
// to the pool when the cached graph that owns it is evicted (cycle_graph records them
// through t_capture_slots); a caller's own capture keeps its slots for the process life.
static std::atomic<uint64_t> g_launch_seq{0};
static std::mutex g_slot_mu;
static std::vector<int> g_graph_free;
static int g_graph_hi = kDirectSlots;
static thread_local std::vector<int>* t_capture_slots = nullptr;

int launch_slot(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
    cudaGetLastError();
    cs = cudaStreamCaptureStatusNone;
  }
  if (cs != cudaStreamCaptureStatusActive)
    return int(g_launch_seq.fetch_add(1, std::memory_order_relaxed) % kDirectSlots);
  std::lock_guard<std::mutex> lk(g_slot_mu);
  int slot = -1;
  if (!g_graph_free.empty()) {
    slot = g_graph_free.back();
    g_graph_free.pop_back();
  } else if (g_graph_hi < kSlots) {
    slot = g_graph_hi++;
  }
  if (slot >= 0 && t_capture_slots) t_capture_slots->push_back(slot);
  return slot;
}

static void release_slots(std::vector<int>& slots) {
  std::lock_guard<std::mutex> lk(g_slot_mu);
  g_graph_free.insert(g_graph_free.end(), slots.begin(), slots.end());
  slots.clear();
}

#include "ps_errsum.cuh"
#include "ps_batch.cuh"
#include "ps_tile.cuh"

static ps_status two_step_impl(const ps_grid* g, const void* uk, const void* ukm1, void* ukp1,
                               const ps_table* t, int64_t lo, int64_t hi, cudaStream_t st,
                               const Halo& h = Halo{}) {
  if (g->dtype == PS_F64) return two_step_f64(g, uk, ukm1, ukp1, t, lo, hi, st, h);
  if (g->arith == PS_ARITH_NATIVE) return two_step_f32n(g, uk, ukm1, ukp1, t, lo, hi, st, h);
  return two_step_f32r(g, uk, ukm1, ukp1, t, lo, hi, st, h);
}

static bool stream_shape(const ps_table* t) {
  return shape_matches<ShapeP5>(t) || shape_matches<ShapeP9>(t) || shape_matches<ShapeC9>(t) ||
         shape_matches<ShapeP13>(t);
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

static ps_status two_step_tb_impl(const ps_grid* g, const void* uk, const void* ukm1, void* op,
                                  void* ol, const ps_table* t, int tsteps, cudaStream_t st,
                                  int64_t lo = 0, int64_t hi = -1, bool rev = false,
                                  int rc = 0, const TBHalo& h = TBHalo{}) {
  if (hi < 0) hi = g->rows;
  if (g->dtype == PS_F64) return tb_f64(g, uk, ukm1, op, ol, t, tsteps, lo, hi, st, rev, rc, h);
  if (g->arith == PS_ARITH_NATIVE)
    return tb_f32n(g, uk, ukm1, op, ol, t, tsteps, lo, hi, st, rev, rc, h);
  return tb_f32r(g, uk, ukm1, op, ol, t, tsteps, lo, hi, st, rev, rc, h);
}

// First step over output rows [lo, hi): two streaming launches for the specialised
// shapes, the runtime-table kernel otherwise (u1 must not alias u0 or v0 for the former).
static ps_status first_step_impl(const ps_grid* g, const void* u0, const void* v0, void* u1,
                                 const ps_table* tu, const ps_table* tv, double tau, int64_t lo,
                                 int64_t hi, cudaStream_t st) {
  const bool per = g->bc == PS_BC_PERIODIC;
  ps_status s = PS_OK;
  if (u1 != u0 && u1 != v0 && stream_shape(tu) && stream_shape(tv) && g->rows >= 4 &&
      g->cols >= 4 && env_int("PS_FORCE_GENERIC", 0) == 0) {
    bool done = false;
    if (g->dtype == PS_F64)
      s = first_f64(g, u0, v0, u1, tu, tv, tau, lo, hi, st, &done);
    else if (g->arith == PS_ARITH_NATIVE)
      s = first_f32n(g, u0, v0, u1, tu, tv, tau, lo, hi, st, &done);
    else
      s = first_f32r(g, u0, v0, u1, tu, tv, tau, lo, hi, st, &done);
    if (done || s != PS_OK) return s;
  }
  if (g->dtype == PS_F64)
    return per ? launch_generic<double, ARITH_REF, true, true>(g, u0, v0, u1, tu, tv, tau, lo, hi, st)
               : launch_generic<double, ARITH_REF, false, true>(g, u0, v0, u1, tu, tv, tau, lo, hi, st);
  if (g->arith == PS_ARITH_NATIVE)
    return per ? launch_generic<float, ARITH_NATIVE, true, true>(g, u0, v0, u1, tu, tv, tau, lo, hi, st)
               : launch_generic<float, ARITH_NATIVE, false, true>(g, u0, v0, u1, tu, tv, tau, lo, hi, st);
  return per ? launch_generic<float, ARITH_REF, true, true>(g, u0, v0, u1, tu, tv, tau, lo, hi, st)
             : launch_generic<float, ARITH_REF, false, true>(g, u0, v0, u1, tu, tv, tau, lo, hi, st);
}

static bool tb_supported(const ps_grid* g, const ps_table* t, int tsteps) {
  const bool shape = shape_matches<ShapeP5>(t) || shape_matches<ShapeP9>(t) ||
                     shape_matches<ShapeC9>(t) || shape_matches<ShapeP13>(t);
  if (!shape || g->rows < 4 || g->cols < 4) return false;
  if (tsteps < 2 || tsteps > 6) return false;
  // depths 5 and 6: shared-product kernels only (f64, radius 1, Dirichlet)
  if (tsteps >= 5 && (PS_TB_SYM == 0 || g->dtype != PS_F64 || table_radius(t) != 1 ||
                      g->bc != PS_BC_DIRICHLET))
    return false;
  // the reference-contract fused kernels share one product per input element and
  // coefficient class (ps_tblock.cuh): the table must give each class one coefficient
  // (every named scheme does); others run unblocked
  const bool ref = g->dtype == PS_F64 || g->arith == PS_ARITH_REF;
  const bool fits = table_radius(t) == 1 || tsteps <= PS_TB_SYM_R2_MAXT;
  const bool sym = PS_TB_SYM == 2   ? (ref && fits)
                   : PS_TB_SYM == 1 ? (g->dtype == PS_F64 && g->bc == PS_BC_DIRICHLET && fits)
                                    : false;
  if (sym) {
    const bool eq = shape_matches<ShapeP5>(t)   ? tb_classes_equal<ShapeP5>(t)
                    : shape_matches<ShapeP9>(t) ? tb_classes_equal<ShapeP9>(t)
                    : shape_matches<ShapeC9>(t) ? tb_classes_equal<ShapeC9>(t)
                                                : tb_classes_equal<ShapeP13>(t);
    if (!eq) return false;
  }
  if (g->bc == PS_BC_DIRICHLET) return true;
  // periodic: images to depth R*tsteps must fit the ghost band, and one wrap (or, for a
  // row slab of a ring, one neighbour's rows) must cover them
  const int64_t D = int64_t(table_radius(t)) * tsteps;
  return D <= g->ghost && D <= g->rows && D <= g->cols;
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
  std::vector<int> slots;  // tile-counter slots its kernel nodes own
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

// Caller holds g_graph_mu and keeps it until the returned exec has been launched (another
// thread could otherwise evict and destroy it between lookup and cudaGraphLaunch).
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
  for (int e = 0; e < g_ngraphs; ++e)
    if (std::memcmp(&g_graphs[e].key, &key, sizeof(key)) == 0) return g_graphs[e].exec;
  cudaStream_t cs = capture_stream(key.dev);
  if (!cs) return nullptr;
  if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  std::vector<int> slots;
  t_capture_slots = &slots;
  int c = cur;
  ps_status st = PS_OK;
  for (int k = 0; k < kGraphCycle && st == PS_OK; ++k) {
    st = two_step_impl(g, lvl[c], lvl[(c + 2) % 3], lvl[(c + 1) % 3], t, 0, g->rows, cs,
                       march_opts(g, k));
    c = (c + 1) % 3;
  }
  t_capture_slots = nullptr;
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(cs, &graph);
  cudaGraphExec_t exec = nullptr;
  if (st != PS_OK || ec != cudaSuccess || !graph ||
      cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    release_slots(slots);
    return nullptr;
  }
  cudaGraphDestroy(graph);
  g_launches.fetch_sub(kGraphCycle, std::memory_order_relaxed);  // captured, not executed
  GraphEntry& slot = g_graphs[g_graph_next];
  if (g_graph_next < g_ngraphs && slot.exec) {
    // an evicted graph may still be executing: its slots go back only once it is destroyed
    // (cudaGraphExecDestroy defers the release until the running launch completes, but the
    // counters must not be handed to a new graph before then)
    cudaDeviceSynchronize();
    cudaGraphExecDestroy(slot.exec);
    release_slots(slot.slots);
  }
  slot.key = key;
  slot.exec = exec;
  slot.slots = std::move(slots);
  g_graph_next = (g_graph_next + 1) % 32;
  g_ngraphs = std::min(g_ngraphs + 1, 32);
  return exec;
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
  return first_step_impl(g, u0, v0, u1, tu, tv, tau, 0, g->rows,
                         static_cast<cudaStream_t>(stream));
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
    std::lock_guard<std::mutex> lk(g_graph_mu);  // held across the launches (see cycle_graph)
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

ps_status ps_two_step_tb_halo(const ps_grid* g, const void* uk, const void* ukm1,
                              void* out_prev, void* out_last, const ps_table* t, int32_t tsteps,
                              int64_t row_lo, int64_t row_hi, void* up_prev, void* up_last,
                              int64_t up_rows, void* dn_prev, void* dn_last, void* stream) {
  ps_status s = check_grid(g);
  if (s != PS_OK) return s;
  if (g->bc != PS_BC_DIRICHLET) return PS_ERR_ARG;
  if (!uk || !ukm1 || !out_prev || !out_last) return PS_ERR_ARG;
  if (out_prev == uk || out_prev == ukm1 || out_last == uk || out_last == ukm1 ||
      out_prev == out_last)
    return PS_ERR_ARG;
  if (row_lo < 0 || row_hi > g->rows || row_lo > row_hi) return PS_ERR_ARG;
  if ((s = check_table(g, t)) != PS_OK) return s;
  if (!tb_supported(g, t, tsteps) || tsteps < 2) return PS_ERR_ARG;
  const int64_t depth = int64_t(table_radius(t)) * tsteps;
  if (depth > g->ghost || depth > g->rows) return PS_ERR_SHAPE;
  if ((up_prev != nullptr) != (up_last != nullptr) || (dn_prev != nullptr) != (dn_last != nullptr))
    return PS_ERR_ARG;
  if (up_prev && up_rows < depth) return PS_ERR_ARG;
  for (const void* q : {uk, ukm1, static_cast<const void*>(out_prev),
                        static_cast<const void*>(out_last), static_cast<const void*>(up_prev),
                        static_cast<const void*>(up_last), static_cast<const void*>(dn_prev),
                        static_cast<const void*>(dn_last)})
    if (q && !aligned16(q)) return PS_ERR_ALIGN;
  TBHalo h;
  h.up_prev = up_prev;
  h.up_last = up_last;
  h.dn_prev = dn_prev;
  h.dn_last = dn_last;
  h.up_rows = int32_t(up_rows);
  return two_step_tb_impl(g, uk, ukm1, out_prev, out_last, t, tsteps,
                          static_cast<cudaStream_t>(stream), row_lo, row_hi, false, 0, h);
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
  if (tsteps < 1 || tsteps > 6) return PS_ERR_ARG;
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

// Tile-resident march (ps_tile.cuh): 1 = this grid / table / depth can run it.
static bool tile_plan_for(const ps_grid* g, const ps_table* t, int tsteps, int* py, int* px,
                          int* th, int* tw, size_t* smem) {
  if (g->dtype != PS_F64 || !single_slab(g)) return false;
  if (tsteps < 1 || tsteps > 16 || !stream_shape(t)) return false;
  const int R = table_radius(t);
  if (g->bc == PS_BC_DIRICHLET && g->ring < R) return false;
  return tile_plan(g->rows, g->cols, R, tsteps, std::max(1, dev_info().nsm),
                   size_t(227) * 1024, py, px, th, tw, smem);
}

int32_t ps_tile_supported(const ps_grid* g, const ps_table* t, int32_t tsteps) {
  if (check_grid(g) != PS_OK || !t || check_table(g, t) != PS_OK) return 0;
  int py, px, th, tw;
  size_t smem;
  return tile_plan_for(g, t, tsteps, &py, &px, &th, &tw, &smem) ? 1 : 0;
}

ps_status ps_march_tile(const ps_grid* g, void* lvl[4], int64_t nsteps, const ps_table* t,
                        int32_t tsteps, int32_t* newest, int32_t* previous, void* stream) {
  ps_status s = check_grid(g);
  if (s != PS_OK) return s;
  if (!lvl || !newest || !previous || nsteps < 0) return PS_ERR_ARG;
  const int cur = *newest, prev = *previous;
  if (cur < 0 || cur > 3 || prev < 0 || prev > 3 || cur == prev) return PS_ERR_ARG;
  for (int x = 0; x < 4; ++x)
    if (!lvl[x] || !aligned16(lvl[x])) return lvl[x] ? PS_ERR_ALIGN : PS_ERR_ARG;
  if ((s = check_table(g, t)) != PS_OK) return s;
  int py, px, th, tw;
  size_t smem;
  if (!tile_plan_for(g, t, tsteps, &py, &px, &th, &tw, &smem)) return PS_ERR_ARG;
  if (nsteps == 0) return PS_OK;
  int f1 = -1, f2 = -1;
  for (int x = 0; x < 4; ++x)
    if (x != cur && x != prev) (f1 < 0 ? f1 : f2) = x;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // epoch flags: one array out of a per-device ring allocated once (a stream-ordered
  // allocation per call cost ~1 ms: the default pool hands its memory back at every
  // synchronisation); 64 marches may be in flight at once before an array is reused
  constexpr int kFlagSets = 64, kFlagStride = 1024;
  static unsigned int* flag_pool[kMaxDevices] = {};
  static std::mutex flag_mu;
  static std::atomic<unsigned> flag_seq{0};
  if (size_t(py) * px > size_t(kFlagStride)) return PS_ERR_ARG;
  unsigned int* flags = nullptr;
  {
    std::lock_guard<std::mutex> lk(flag_mu);
    const int dev = device_index();
    if (!flag_pool[dev] &&
        cudaMalloc(reinterpret_cast<void**>(&flag_pool[dev]),
                   sizeof(unsigned int) * kFlagSets * kFlagStride) != cudaSuccess)
      return PS_ERR_CUDA;
    flags = flag_pool[dev] + size_t(flag_seq.fetch_add(1) % kFlagSets) * kFlagStride;
  }
#define PS_TILE_GO(S)                                                                          \
  (g->bc == PS_BC_PERIODIC                                                                     \
       ? launch_tile<S, true>(g, lvl, nsteps, t, tsteps, cur, prev, f1, f2, flags, st, py, px, \
                              th, tw, smem)                                                    \
       : launch_tile<S, false>(g, lvl, nsteps, t, tsteps, cur, prev, f1, f2, flags, st, py,    \
                               px, th, tw, smem))
  if (shape_matches<ShapeP5>(t))
    s = PS_TILE_GO(ShapeP5);
  else if (shape_matches<ShapeP9>(t))
    s = PS_TILE_GO(ShapeP9);
  else if (shape_matches<ShapeC9>(t))
    s = PS_TILE_GO(ShapeC9);
  else
    s = PS_TILE_GO(ShapeP13);
#undef PS_TILE_GO
  if (s != PS_OK) return s;
  const int64_t nepochs = (nsteps + tsteps - 1) / tsteps;
  if (nepochs & 1) {
    *newest = f2;
    *previous = f1;
  }
  if (g->bc == PS_BC_PERIODIC) {
    // the tiles wrote the n x n cores only: refresh the images other kernels read
    if ((s = ps_fill_ghosts(g, lvl[*newest], 0, stream)) != PS_OK) return s;
    if ((s = ps_fill_ghosts(g, lvl[*previous], 0, stream)) != PS_OK) return s;
  }
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
  k_errsum_leaves<<<unsigned((int64_t(p.nleaves) * 8 + 255) / 256), 256, 0, st_>>>(
      at_origin<double>(g, level), at_origin<double>(g, S), g->pitch, p.cols_h, st,
      p.leaf_start, p.leaf_len, p.nleaves, p.values, nvalues);
  k_errsum_fold<<<1, 1024, 0, st_>>>(p.node_left, p.node_right, p.node_id, p.level_off,
                                      p.nlevels, p.values, nvalues, p.root, out2);
  g_launches.fetch_add(2, std::memory_order_relaxed);
  return last_cuda_status();
}

ps_status ps_march_errsum(const ps_grid* g, void* lvl[3], int64_t nsteps, const ps_table* t,
                          ps_errsum* e, const void* S, const double* st_host, double* out_dev,
                          int32_t* newest, void* stream) {
  // run()'s loop (simulator.py:271-280) without a host round trip per step: each
  // two-step update is followed by its error sums, written to out_dev[2k], out_dev[2k+1].
  if (!e || !S || !st_host || !out_dev || !lvl || !newest || nsteps < 0) return PS_ERR_ARG;
  for (int64_t k = 0; k < nsteps; ++k) {
    ps_status s = ps_march(g, lvl, 1, t, newest, stream);
    if (s != PS_OK) return s;
    if ((s = ps_errsum_step(e, g, lvl[*newest], S, st_host[k], out_dev + 2 * k, stream)) != PS_OK)
      return s;
  }
  return PS_OK;
}

static bool batch_table(ps::BatchTable& d, const ps_table& t) {
  if (t.ntaps < 1 || t.ntaps > PS_MAX_TAPS) return false;
  d.n = t.ntaps;
  for (int s = 0; s < t.ntaps; ++s) {
    if (t.q1[s] < -100 || t.q1[s] > 100 || t.q2[s] < -100 || t.q2[s] > 100) return false;
    d.q1[s] = int8_t(t.q1[s]);
    d.q2[s] = int8_t(t.q2[s]);
    d.c[s] = t.c[s];
  }
  return true;
}

size_t ps_batch_desc_bytes(void) { return sizeof(ps::BatchDev); }

ps_status ps_batch_pack(const ps_batch_sim* sim, void* desc_host) {
  if (!sim || !desc_host) return PS_ERR_ARG;
  if (sim->n < 2 || sim->n > PS_BATCH_MAX_N || sim->n_t < 1) return PS_ERR_SHAPE;
  if (sim->bc != PS_BC_DIRICHLET && sim->bc != PS_BC_PERIODIC) return PS_ERR_ARG;
  ps::BatchDev d;
  std::memset(&d, 0, sizeof(d));
  d.n = sim->n;
  d.nt = sim->n_t;
  d.bc = sim->bc;
  d.tau = sim->tau;
  if (!batch_table(d.tu, sim->first_u) || !batch_table(d.tv, sim->first_v) ||
      !batch_table(d.t2, sim->two_step))
    return PS_ERR_TABLE;
  d.off_field = sim->off_field;
  d.off_st = sim->off_st;
  d.off_out = sim->off_out;
  std::memcpy(desc_host, &d, sizeof(d));
  return PS_OK;
}

ps_status ps_batch_run(int32_t nsim, int32_t max_n, const void* desc_dev, const double* u0,
                       const double* v0, const double* S, const double* st, double* out,
                       void* stream) {
  if (nsim < 1 || !desc_dev || !u0 || !v0 || !S || !st || !out) return PS_ERR_ARG;
  if (max_n < 2 || max_n > PS_BATCH_MAX_N) return PS_ERR_SHAPE;
  const size_t nn = size_t(max_n + 1) * size_t(max_n + 1);
  const size_t smem = 3 * nn * sizeof(double) + 4 * ps::kBatchMaxLeaves * sizeof(double) +
                      (4 * ps::kBatchMaxLeaves + 2) * sizeof(int);
  static std::once_flag once[ps::kMaxDevices];  // per-device function attribute
  std::call_once(once[ps::device_index()], [] {
    cudaFuncSetAttribute(ps::k_batch_run, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
  });
  if (smem > 227 * 1024) return PS_ERR_SHAPE;
  ps::k_batch_run<<<unsigned(nsim), ps::kBatchThreads, smem, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const ps::BatchDev*>(desc_dev), u0, v0, S, st, out);
  g_launches.fetch_add(1, std::memory_order_relaxed);
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

#include "ps_solve.cuh"
