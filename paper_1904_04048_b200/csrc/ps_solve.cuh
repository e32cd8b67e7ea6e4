// ps_solve.cuh — host-to-host solve with the PCIe copies hidden behind the march
// (ps_solve_plan / ps_solve_host in include/ps.h).  Included at the end of ps_device.cu.
//
// Why: the drop-in's end-to-end path starts from host arrays (the reference's run() samples
// u0/v0 on the host, simulator.py:253-270) and ends with a host array.  Copying a whole
// level in, marching, and copying it out serialises ~2 x 8.6 GB of PCIe traffic (~330 ms
// on C4) with ~470 ms of stencil work.  Row bands marched as a skewed wavefront let band b
// run all of its launches while band b+1 is still uploading and band b-1 downloads.
//
// Plan (Dirichlet; rows do not wrap).  Band b owns rows [S_b, S_{b+1}), S_b = b*H, the
// last band reaching past the grid.  Its launch j (j = 0 the first step, then fused passes
// of T updates, then single-update tail steps — the launches ps_march_tb would issue)
// writes rows [S_b - o_j, S_{b+1} - o_j) with o_j = s*(j+1), s = R*T_max >= every
// launch's read reach.  Then
//   * rows launch j of band b reads above its range (>= S_b - o_j - s) hold launch j-1's
//     output there: band b-1's launch j-1 wrote up to S_b - o_{j-1}, and band b-1's
//     launches >= j+1 only write below S_b - o_{j+1} = S_b - o_j - s (bands are at
//     least 2s rows tall, so those rows lie in band b-1's range);
//   * rows it reads below its range come from band b's own launch j-1;
//   * so launch (b, j) needs (b, j-1) and (b-1, j-1) — nothing else — and band b-1 may
//     run ahead of band b; each launch's outputs never alias the inputs it reads at
//     neighbour rows (fused passes and tail steps write free levels; the first step's
//     second half reads u1 only at its own rows).
// The compute launches alternate between `nstreams` streams by band, so a band's tail
// wave overlaps the next band's launches; uploads and downloads have their own streams.
#pragma once

namespace ps {

struct SolvePlanIn {
  int64_t rows = 0;
  int radius = 1;
  int64_t nsteps = 1;
  int tsteps = 1;
  int nbands = 0;
  int nstreams = 2;
};

static int64_t solve_auto_bands(int64_t rows, int s) {
  // about 1024 rows per band (C4 sweep, profiles/r01_solve_tune_c4.jsonl: 16 bands 461,
  // 32 bands 468 GLUP/s host-to-host; the fill and drain shrink with the band)
  int64_t B = (rows + 512) / 1024;
  B = std::min<int64_t>(B, 64);
  B = std::min<int64_t>(B, rows / std::max<int64_t>(1, 8 * s));  // bands >= 8 skews tall
  return std::max<int64_t>(B, 1);
}

static ps_status build_solve_plan(const SolvePlanIn& in, std::vector<ps_solve_op>& ops) {
  ops.clear();
  if (in.rows < 1 || in.radius < 0 || in.nsteps < 1) return PS_ERR_ARG;
  if (in.tsteps < 1 || in.tsteps > 6) return PS_ERR_ARG;
  if (in.nstreams < 1 || in.nstreams > 8 || in.nbands < 0) return PS_ERR_ARG;
  const int T = in.tsteps;
  const int64_t m = in.nsteps - 1;                    // two-step updates after the first step
  const int64_t npass = T > 1 ? m / T : 0;
  const int64_t ntail = m - npass * T;
  const int64_t J = 1 + npass + ntail;                // compute launches per band
  const int64_t s = std::max<int64_t>(1, int64_t(in.radius) * T);
  int64_t B = in.nbands > 0 ? in.nbands : solve_auto_bands(in.rows, int(s));
  // launch j reads at most s rows above its range start S_b - o_j; band b-1's launch j-1
  // starts at S_b - H - o_j + s, so bands at least 2s tall keep those rows inside band
  // b-1 (the only band ordered before it)
  B = std::max<int64_t>(1, std::min<int64_t>(B, in.rows / (2 * s)));
  const int64_t H = (in.rows + B - 1) / B;
  B = (in.rows + H - 1) / H;
  const int64_t far = in.rows + s * (J + 1);          // end of the last band
  auto S = [&](int64_t b) { return b >= B ? far : b * H; };
  const int store_stream = in.nstreams + 1;
  ops.reserve(size_t(B * (J + 2)));
  std::vector<int64_t> prev_band(size_t(J), -1), cur_band(size_t(J), -1);
  for (int64_t b = 0; b < B; ++b) {
    ps_solve_op ld{};
    ld.kind = PS_OP_LOAD;
    ld.band = int32_t(b);
    ld.stream = 0;
    ld.src0 = ld.src1 = -1;
    ld.dst0 = 0;  // u0
    ld.dst1 = 2;  // v0
    ld.row_lo = S(b);
    ld.row_hi = std::min(S(b + 1), in.rows);
    ld.after0 = ld.after1 = -1;
    const int64_t load_idx = int64_t(ops.size());
    ops.push_back(ld);
    const int cstream = 1 + int(b % in.nstreams);
    int cur = 1, prev = 0;  // after the first step: u1 in level 1, u0 in level 0
    for (int64_t j = 0; j < J; ++j) {
      ps_solve_op op{};
      op.band = int32_t(b);
      op.stream = cstream;
      const int64_t o = s * (j + 1);
      op.row_lo = std::max<int64_t>(0, S(b) - o);
      op.row_hi = std::max(op.row_lo, std::min(in.rows, S(b + 1) - o));
      op.after0 = j == 0 ? load_idx : -1;
      op.after1 = (b > 0 && j > 0) ? prev_band[size_t(j - 1)] : -1;
      op.dst0 = -1;
      int f1 = -1, f2 = -1;
      for (int x = 0; x < 4; ++x)
        if (x != cur && x != prev) (f1 < 0 ? f1 : f2) = x;
      if (j == 0) {
        op.kind = PS_OP_FIRST;
        op.tsteps = 1;
        op.src0 = 0;
        op.src1 = 2;
        op.dst1 = 1;
      } else if (j <= npass) {
        op.kind = PS_OP_PASS;
        op.tsteps = T;
        op.src0 = cur;
        op.src1 = prev;
        op.dst0 = f1;
        op.dst1 = f2;
        prev = f1;
        cur = f2;
      } else {
        op.kind = PS_OP_STEP;
        op.tsteps = 1;
        op.src0 = cur;
        op.src1 = prev;
        op.dst1 = f1;
        prev = cur;
        cur = f1;
      }
      cur_band[size_t(j)] = int64_t(ops.size());
      ops.push_back(op);
    }
    ps_solve_op st{};
    st.kind = PS_OP_STORE;
    st.band = int32_t(b);
    st.stream = store_stream;
    st.src0 = cur;
    st.src1 = st.dst0 = st.dst1 = -1;
    const int64_t o = s * J;
    st.row_lo = std::max<int64_t>(0, S(b) - o);
    st.row_hi = std::max(st.row_lo, std::min(in.rows, S(b + 1) - o));
    st.after0 = cur_band[size_t(J - 1)];
    st.after1 = -1;
    ops.push_back(st);
    std::swap(prev_band, cur_band);
  }
  return PS_OK;
}

// Copy host rows [lo, hi) (row stride hp elements) into / out of a level's logical block.
static cudaError_t rows_copy(const ps_grid* g, void* level, const void* host, int64_t hp,
                             int64_t lo, int64_t hi, int64_t cols_h, bool in, cudaStream_t st) {
  if (hi <= lo) return cudaSuccess;
  const size_t esz = g->dtype == PS_F64 ? 8 : 4;
  char* dev = static_cast<char*>(level) + (g->origin + lo * g->pitch) * esz;
  const char* h = static_cast<const char*>(host) + lo * hp * esz;
  if (in)
    return cudaMemcpy2DAsync(dev, g->pitch * esz, h, hp * esz, cols_h * esz, size_t(hi - lo),
                             cudaMemcpyHostToDevice, st);
  return cudaMemcpy2DAsync(const_cast<char*>(h), hp * esz, dev, g->pitch * esz, cols_h * esz,
                           size_t(hi - lo), cudaMemcpyDeviceToHost, st);
}

// Streams and events of one ps_solve_host call (released when the call returns; CUDA
// defers the destruction until the queued work completes).
struct SolveRes {
  std::vector<cudaStream_t> own;
  std::vector<cudaEvent_t> ev;
  ~SolveRes() {
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
    for (cudaStream_t s : own)
      if (s) cudaStreamDestroy(s);
  }
};

}  // namespace ps

extern "C" {

int64_t ps_solve_plan(int64_t rows, int32_t radius, int64_t nsteps, int32_t tsteps,
                      int32_t nbands, int32_t nstreams, ps_solve_op* ops, int64_t max_ops) {
  ps::SolvePlanIn in;
  in.rows = rows;
  in.radius = radius;
  in.nsteps = nsteps;
  in.tsteps = tsteps;
  in.nbands = nbands;
  in.nstreams = nstreams;
  std::vector<ps_solve_op> plan;
  const ps_status s = ps::build_solve_plan(in, plan);
  if (s != PS_OK) return -int64_t(s);
  if (ops)
    for (int64_t i = 0; i < std::min<int64_t>(max_ops, int64_t(plan.size())); ++i) ops[i] = plan[size_t(i)];
  return int64_t(plan.size());
}

ps_status ps_solve_host(const ps_grid* g, void* lvl[4], const void* u0_host,
                        const void* v0_host, void* out_host, int64_t host_pitch,
                        const ps_table* tu, const ps_table* tv, const ps_table* t, double tau,
                        int64_t nsteps, int32_t tsteps, int32_t nbands, void* stream) {
  using namespace ps;
  ps_status s = check_grid(g);
  if (s != PS_OK) return s;
  if (!lvl || !u0_host || !out_host || nsteps < 1 || nbands < 0) return PS_ERR_ARG;
  if (tsteps < 1 || tsteps > 6) return PS_ERR_ARG;
  for (int x = 0; x < 4; ++x) {
    if (!lvl[x]) return PS_ERR_ARG;
    if (!aligned16(lvl[x])) return PS_ERR_ALIGN;
    for (int y = 0; y < x; ++y)
      if (lvl[x] == lvl[y]) return PS_ERR_ARG;
  }
  if ((s = check_table(g, tu)) != PS_OK || (s = check_table(g, tv)) != PS_OK ||
      (s = check_table(g, t)) != PS_OK)
    return s;
  if (!single_slab(g)) return PS_ERR_SHAPE;
  const bool per = g->bc == PS_BC_PERIODIC;
  const int64_t a = per ? 1 : 0;  // the reference's alias row / column
  const int64_t rows_h = g->rows + a, cols_h = g->cols + a;
  if (host_pitch < cols_h) return PS_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (tsteps > 1 && !tb_supported(g, t, tsteps)) tsteps = 1;

  if (per) {
    // rows wrap: one band — upload, march, download on the caller's stream
    const int kind_in = 1, kind_out = 2;
    if ((s = ps_copy_in(g, lvl[0], u0_host, rows_h, cols_h, host_pitch, kind_in, stream)) != PS_OK)
      return s;
    if (v0_host) {
      if ((s = ps_copy_in(g, lvl[2], v0_host, rows_h, cols_h, host_pitch, kind_in, stream)) != PS_OK)
        return s;
    } else if (cudaMemsetAsync(lvl[2], 0, ps_level_bytes(g), st) != cudaSuccess) {
      return PS_ERR_CUDA;
    }
    if ((s = ps_fill_ghosts(g, lvl[0], 0, stream)) != PS_OK) return s;
    if ((s = ps_fill_ghosts(g, lvl[2], 0, stream)) != PS_OK) return s;
    if ((s = first_step_impl(g, lvl[0], lvl[2], lvl[1], tu, tv, tau, 0, g->rows, st)) != PS_OK)
      return s;
    int32_t cur = 1, prev = 0;
    bool tiled = false;
    if (env_int("PS_SOLVE_TILE", 1) != 0 && nsteps > 1 && nbands == 0) {
      // small grids: all the updates in one tile-resident launch (ps_march_tile)
      for (const int depth : {12, 8, 4}) {
        int py, px, th, tw;
        size_t smem;
        if (!tile_plan_for(g, t, depth, &py, &px, &th, &tw, &smem)) continue;
        if ((s = ps_march_tile(g, lvl, nsteps - 1, t, depth, &cur, &prev, stream)) != PS_OK)
          return s;
        tiled = true;
        break;
      }
    }
    if (!tiled &&
        (s = ps_march_tb(g, lvl, nsteps - 1, t, tsteps, &cur, &prev, stream)) != PS_OK)
      return s;
    return ps_copy_out(g, lvl[cur], out_host, rows_h, cols_h, host_pitch, kind_out, stream);
  }

  // small Dirichlet f64 grids (a level of a few MB: the reference's own sizes): no bands --
  // upload, first step, the tile-resident march (ps_march_tile: one cooperative launch for
  // all nsteps - 1 updates), download.  C1 (512^2, 200 steps): 2.7 ms -> see DESIGN.md §9.
  // (only when the caller leaves the banding to the library: an explicit nbands keeps the
  // banded wavefront, which is how the tests drive it on small grids)
  if (env_int("PS_SOLVE_TILE", 1) != 0 && nsteps > 1 && nbands == 0 &&
      env_int("PS_SOLVE_BANDS", 0) == 0) {
    for (const int depth : {12, 8, 4}) {
      int py, px, th, tw;
      size_t smem;
      if (!tile_plan_for(g, t, depth, &py, &px, &th, &tw, &smem)) continue;
      if ((s = ps_copy_in(g, lvl[0], u0_host, rows_h, cols_h, host_pitch, 1, stream)) != PS_OK)
        return s;
      if (v0_host) {
        if ((s = ps_copy_in(g, lvl[2], v0_host, rows_h, cols_h, host_pitch, 1, stream)) != PS_OK)
          return s;
      } else if (cudaMemsetAsync(lvl[2], 0, ps_level_bytes(g), st) != cudaSuccess) {
        return PS_ERR_CUDA;
      }
      if ((s = first_step_impl(g, lvl[0], lvl[2], lvl[1], tu, tv, tau, 0, g->rows, st)) != PS_OK)
        return s;
      int32_t cur = 1, prev = 0;
      if ((s = ps_march_tile(g, lvl, nsteps - 1, t, depth, &cur, &prev, stream)) != PS_OK)
        return s;
      return ps_copy_out(g, lvl[cur], out_host, rows_h, cols_h, host_pitch, 2, stream);
    }
  }

  SolvePlanIn in;
  in.rows = g->rows;
  in.radius = std::max(table_radius(t), std::max(table_radius(tu), table_radius(tv)));
  in.nsteps = nsteps;
  in.tsteps = tsteps;
  in.nbands = env_int("PS_SOLVE_BANDS", nbands);
  // three compute streams: with the 672-column strips of the shared-product kernel a
  // 1024-row band is 1.3 waves of tiles, and a third stream keeps the tail of one band's
  // launch covered (C4, 200 steps: 395-400 ms for 16-48 bands; two streams 403-479 ms;
  // profiles/r02_solve_tune_c4.jsonl)
  in.nstreams = std::max(1, std::min(8, env_int("PS_SOLVE_STREAMS", 3)));
  std::vector<ps_solve_op> plan;
  if ((s = build_solve_plan(in, plan)) != PS_OK) return s;
  // fused passes in bands: taller tiles than the whole-grid heuristic picks for a short
  // launch (fewer recomputed halo rows; the next band's launch fills the tail)
  const int rc = env_int("PS_SOLVE_RC", 256);

  SolveRes res;
  const int nstreams_total = in.nstreams + 2;
  std::vector<cudaStream_t> ss(size_t(nstreams_total), nullptr);
  for (int x = 0; x < nstreams_total; ++x) {
    if (x == 1) {
      ss[1] = st;
      continue;
    }
    cudaStream_t ns = nullptr;
    if (cudaStreamCreateWithFlags(&ns, cudaStreamNonBlocking) != cudaSuccess) return PS_ERR_CUDA;
    res.own.push_back(ns);
    ss[size_t(x)] = ns;
  }
  // event ring: op i's event is re-recorded by op i + ring, after its last waiter issued
  int64_t ring = 1;
  for (int64_t i = 0; i < int64_t(plan.size()); ++i)
    for (int64_t w : {plan[size_t(i)].after0, plan[size_t(i)].after1})
      if (w >= 0) ring = std::max(ring, i - w + 1);
  res.ev.assign(size_t(ring + 1 + nstreams_total), nullptr);
  for (auto& e : res.ev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return PS_ERR_CUDA;
  cudaEvent_t start = res.ev[size_t(ring)];
  if (cudaEventRecord(start, st) != cudaSuccess) return PS_ERR_CUDA;
  for (int x = 0; x < nstreams_total; ++x)
    if (x != 1 && cudaStreamWaitEvent(ss[size_t(x)], start, 0) != cudaSuccess) return PS_ERR_CUDA;

  const size_t esz = g->dtype == PS_F64 ? 8 : 4;
  for (int64_t i = 0; i < int64_t(plan.size()); ++i) {
    const ps_solve_op& op = plan[size_t(i)];
    cudaStream_t os = ss[size_t(op.stream)];
    for (int64_t w : {op.after0, op.after1})
      if (w >= 0 && cudaStreamWaitEvent(os, res.ev[size_t(w % ring)], 0) != cudaSuccess)
        return PS_ERR_CUDA;
    const int64_t lo = op.row_lo, hi = op.row_hi;
    switch (op.kind) {
      case PS_OP_LOAD:
        if (rows_copy(g, lvl[op.dst0], u0_host, host_pitch, lo, hi, cols_h, true, os) != cudaSuccess)
          return PS_ERR_CUDA;
        if (v0_host) {
          if (rows_copy(g, lvl[op.dst1], v0_host, host_pitch, lo, hi, cols_h, true, os) != cudaSuccess)
            return PS_ERR_CUDA;
        } else if (hi > lo) {
          char* d = static_cast<char*>(lvl[op.dst1]) + (g->origin + lo * g->pitch) * esz;
          if (cudaMemset2DAsync(d, g->pitch * esz, 0, g->cols * esz, size_t(hi - lo), os) !=
              cudaSuccess)
            return PS_ERR_CUDA;
        }
        break;
      case PS_OP_FIRST:
        s = first_step_impl(g, lvl[op.src0], lvl[op.src1], lvl[op.dst1], tu, tv, tau, lo, hi, os);
        break;
      case PS_OP_STEP:
        s = two_step_impl(g, lvl[op.src0], lvl[op.src1], lvl[op.dst1], t, lo, hi, os);
        break;
      case PS_OP_PASS:
        s = two_step_tb_impl(g, lvl[op.src0], lvl[op.src1], lvl[op.dst0], lvl[op.dst1], t,
                             op.tsteps, os, lo, hi, false, rc);
        break;
      case PS_OP_STORE:
        if (rows_copy(g, lvl[op.src0], out_host, host_pitch, lo, hi, cols_h, false, os) !=
            cudaSuccess)
          return PS_ERR_CUDA;
        break;
      default:
        return PS_ERR_ARG;
    }
    if (s != PS_OK) return s;
    if (cudaEventRecord(res.ev[size_t(i % ring)], os) != cudaSuccess) return PS_ERR_CUDA;
  }
  // the caller's stream resumes after every side stream's work
  for (int x = 0; x < nstreams_total; ++x) {
    if (x == 1) continue;
    cudaEvent_t e = res.ev[size_t(ring + 1 + x)];
    if (cudaEventRecord(e, ss[size_t(x)]) != cudaSuccess || cudaStreamWaitEvent(st, e, 0) != cudaSuccess)
      return PS_ERR_CUDA;
  }
  return PS_OK;
}

}  // extern "C"
