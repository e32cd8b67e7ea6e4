/*
 * ps.h — C-ABI of libps.so, the B200 (sm_100a) engine behind the poisson_stencils
 * drop-in.  Plain pointers and sizes only; no torch or numpy types cross this line.
 *
 * The reference (poisson-stencils 0.1.0, pure Python/numpy) has no FFI.  Each entry
 * point below replaces one reference function; the citation names the file:line of the
 * function it stands in for (paths relative to the reference's pkg/src/poisson_stencils/).
 * INTEGRATION.md shows the ctypes binding a maintainer adds on the reference side.
 *
 * Conventions
 *   - Field pointers ("levels") are DEVICE pointers to an allocation laid out by
 *     ps_layout_init(): logical element (i, j) lives at  level[grid->origin + i*pitch + j].
 *     Around the logical rows x cols block the allocation holds `ghost` padding rows above
 *     and below and >= 16 bytes of padding columns on each side.  Periodic grids keep
 *     their wrap-around images (rows/cols -ghost..-1 and n..n+ghost-1) in that padding;
 *     every kernel that writes a periodic level also refreshes its images.
 *   - Logical extent: Dirichlet grids hold all (n+1) x (n+1) nodes (ring included);
 *     periodic grids hold the n x n independent nodes; the reference's alias row/col n
 *     is the first image row/col.
 *   - Calls are asynchronous on the given stream (NULL = legacy default stream), never
 *     allocate device memory, and are safe from concurrent threads and streams.  The only
 *     library state is a mutex-guarded cache of instantiated CUDA graphs (ps_march; the
 *     lock is held until a cached graph has been launched, so no thread can evict it in
 *     between) and the tile counters of the streaming kernels: every direct launch takes
 *     the next of 2048 counter slots (so fewer than 2048 launches of this library may be
 *     in flight at once), every kernel node of a captured CUDA graph — ps_march's own or a
 *     caller's stream capture around these calls — owns a slot of a separate pool of 2048
 *     for the life of the graph (PS_ERR_CUDA once that pool is exhausted).
 *   - Return 0 (PS_OK) or a distinct ps_status; ps_strerror() names it.
 */
#ifndef PS_H_
#define PS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum ps_status {
  PS_OK = 0,
  PS_ERR_ARG = 1,        /* bad argument (null pointer, bad enum, negative size)          */
  PS_ERR_SHAPE = 2,      /* grid too small for the stencil / layout mismatch              */
  PS_ERR_TABLE = 3,      /* coefficient table empty, too long or offsets beyond the ghost */
  PS_ERR_RADIUS = 4,     /* Dirichlet ring narrower than the stencil radius (cli.py:24)   */
  PS_ERR_CUDA = 5,       /* a CUDA runtime call failed                                    */
  PS_ERR_ALIGN = 6       /* level pointer not 16-byte aligned                             */
} ps_status;

typedef enum ps_bc { PS_BC_DIRICHLET = 0, PS_BC_PERIODIC = 1 } ps_bc;
typedef enum ps_dtype { PS_F64 = 0, PS_F32 = 1 } ps_dtype;

/* Arithmetic contract.
 *   PS_ARITH_REF    — the reference's own operation sequence, bit for bit (simulator.py:147-191):
 *                     f64: acc = +0.0; acc = fl(acc + fl(c*u)) in table order, no FMA;
 *                     f32: products in f32, accumulation in f64, cast to f32, f32 subtract.
 *   PS_ARITH_NATIVE — f32 only: taps in the same table order folded with one correctly
 *                     rounded fma each (acc = fma(c, u, acc) from +0.0, f32 accumulator),
 *                     then an f32 subtract.  Bitwise against the oracle's fmaf() chain;
 *                     against the f64 run within a stated tolerance.  f64: same as REF. */
typedef enum ps_arith { PS_ARITH_REF = 0, PS_ARITH_NATIVE = 1 } ps_arith;

#define PS_MAX_TAPS 32
#define PS_MAX_GHOST 8

/* One coefficient table evaluated at the Courant number, in the reference's dict order
 * (scheme.py:26-51 tables, evaluated by simulator.py:131-132 -> quadrature.py:107-108).
 * Tap s reads u[i + q1[s], j + q2[s]] (q1 along axis 0 = x1, q2 along axis 1 = x2). */
typedef struct ps_table {
  int32_t ntaps;
  int32_t q1[PS_MAX_TAPS];
  int32_t q2[PS_MAX_TAPS];
  double c[PS_MAX_TAPS];
} ps_table;

/* Geometry and numerics of one family of levels; filled by ps_layout_init(). */
typedef struct ps_grid {
  int64_t rows;    /* logical rows  (Dirichlet n+1, periodic n)             */
  int64_t cols;    /* logical cols                                          */
  int64_t pitch;   /* elements between consecutive rows (multiple of 128 B) */
  int64_t origin;  /* element offset of logical (0,0) from the allocation   */
  int64_t ghost;   /* padding rows above/below the logical block            */
  int64_t row0;    /* global index of logical row 0 (row slabs; else 0)     */
  int64_t grows;   /* global logical rows (row slabs; else == rows)         */
  int32_t ring;    /* Dirichlet: width of the pinned zero ring; periodic: 0 */
  int32_t bc;      /* ps_bc    */
  int32_t dtype;   /* ps_dtype */
  int32_t arith;   /* ps_arith */
} ps_grid;

/* Fill *g for a rows x cols grid.  `ghost` = largest stencil radius the levels must
 * serve (>= 1; rounded up to 2).  `ring` = Dirichlet ring width (ignored for periodic).
 * Replaces the implicit layout of numpy arrays allocated per step (simulator.py:150). */
ps_status ps_layout_init(ps_grid* g, int64_t rows, int64_t cols, int32_t ghost, int32_t ring,
                         int32_t bc, int32_t dtype, int32_t arith);
/* Row slab of a global grid for the multi-GPU decomposition: the
 * level holds global rows [row0, row0 + rows) as logical rows 0..rows-1; its `ghost`
 * padding rows receive the neighbours' halo rows (global rows row0-ghost.. and
 * row0+rows..).  Dirichlet ring masking uses global indices against `grows`.
 * Periodic slabs wrap columns locally and rows through the halo exchange. */
ps_status ps_slab_layout_init(ps_grid* g, int64_t grows, int64_t cols, int64_t row0,
                              int64_t rows, int32_t ghost, int32_t ring, int32_t bc,
                              int32_t dtype, int32_t arith);

/* Bytes one level of *g occupies. */
size_t ps_level_bytes(const ps_grid* g);

/* Convenience allocation for callers without their own allocator (ctypes users).
 * The level is zero-filled.  Returns NULL on failure. */
void* ps_level_alloc(const ps_grid* g);
void ps_level_free(void* level);

/* Copy a dense host/device rows_h x cols_h block (row stride host_pitch elements) into /
 * out of the logical block of a level, starting at logical (0,0).  rows_h/cols_h may
 * exceed rows/cols by up to `ghost` for periodic grids (the reference's alias row/col).
 * `kind`: cudaMemcpyKind value (1 = H2D, 2 = D2H, 3 = D2D, 4 = default). */
ps_status ps_copy_in(const ps_grid* g, void* level, const void* src, int64_t rows_h,
                     int64_t cols_h, int64_t src_pitch, int32_t kind, void* stream);
ps_status ps_copy_out(const ps_grid* g, const void* level, void* dst, int64_t rows_h,
                      int64_t cols_h, int64_t dst_pitch, int32_t kind, void* stream);

/* Periodic: refresh every image position from the core (simulator.py:135-138,
 * _alias_edges).  keep_alias != 0 leaves the reference's alias row n / col n
 * (0 <= i,j <= n) untouched, so a caller-supplied u^{k-1} alias survives (simulator.py:184).
 * Dirichlet: no-op. */
ps_status ps_fill_ghosts(const ps_grid* g, void* level, int32_t keep_alias, void* stream);

/* First time step  u1 = A_u(u0) + fl(tau * A_v(v0))  (simulator.py:166-180, run() 269-270). */
ps_status ps_first_step(const ps_grid* g, const void* u0, const void* v0, void* u1,
                        const ps_table* tu, const ps_table* tv, double tau, void* stream);

/* Two-step update  u^{k+1} = A(u^k) - u^{k-1}, ring re-pinned / images refreshed
 * (simulator.py:183-205).  ukp1 must not alias uk; it MAY alias ukm1 (each point of
 * u^{k-1} is read only by the thread that overwrites it). */
ps_status ps_two_step(const ps_grid* g, const void* uk, const void* ukm1, void* ukp1,
                      const ps_table* t, void* stream);

/* ps_two_step restricted to logical rows [row_lo, row_hi): lets a slab update its
 * boundary rows first, hand them to the halo exchange, and update the interior
 * concurrently. */
ps_status ps_two_step_rows(const ps_grid* g, const void* uk, const void* ukm1, void* ukp1,
                           const ps_table* t, int64_t row_lo, int64_t row_hi, void* stream);

/* Row-slab update with in-kernel halo delivery (the fused variant):
 * as ps_two_step_rows, and the CTAs that write the first / last R rows also store them
 * straight into the neighbour slabs' ghost rows — `up_ukp1` (the u^{k+1} level of the
 * slab above, whose logical rows number `up_rows`) receives rows [0,R) at its rows
 * [up_rows, up_rows+R); `dn_ukp1` (slab below) receives rows [rows-R, rows) at its rows
 * [-R, 0).  Peer pointers are allocation bases (as from ps_ipc_open) on any device
 * reachable by peer access (NVLink); NULL = no neighbour.  Dirichlet slabs only.  The
 * caller orders the next step after the neighbours' launches (event / NCCL token). */
ps_status ps_two_step_halo(const ps_grid* g, const void* uk, const void* ukm1, void* ukp1,
                           const ps_table* t, int64_t row_lo, int64_t row_hi, void* up_ukp1,
                           int64_t up_rows, void* dn_ukp1, void* stream);

/* CUDA IPC plumbing for peer levels across processes (64-byte opaque handles).
 * ps_ipc_get_handle names the allocation containing dev_ptr and returns dev_ptr's byte
 * offset in it; the receiver adds that offset to the pointer ps_ipc_open returns. */
ps_status ps_ipc_get_handle(const void* dev_ptr, void* handle64, int64_t* offset);
ps_status ps_ipc_open(const void* handle64, void** dev_ptr);
ps_status ps_ipc_close(void* dev_ptr);

/* nsteps two-step updates rotating three levels in place (the loop of run(),
 * simulator.py:271-274).  On entry lvl[*newest] = u^k and lvl[(*newest+2)%3] = u^{k-1};
 * on return *newest names the level holding the last update.  For nsteps >= 12 six
 * launches (two rotation cycles) are captured into a CUDA graph once per (grid, levels,
 * table, phase) and replayed (environment PS_GRAPH=0 disables); odd steps on grids of
 * <= 256 MB per level walk their tiles bottom-up to reuse the previous step's L2 lines. */
ps_status ps_march(const ps_grid* g, void* lvl[3], int64_t nsteps, const ps_table* t,
                   int32_t* newest, void* stream);

/* Temporal blocking: tsteps (2..4; 5 and 6 for f64 radius-1 Dirichlet tables) updates fused into one
 * streaming pass over u^k / u^{k-1}; writes only u^{k+tsteps-1} (out_prev) and
 * u^{k+tsteps} (out_last).  HBM traffic 4/tsteps words per update instead of 3.
 * Dirichlet grids, shapes P5/P9/C9/P13; results bitwise equal to tsteps ps_two_step
 * calls.  The four buffers must be distinct. */
ps_status ps_two_step_tb(const ps_grid* g, const void* uk, const void* ukm1, void* out_prev,
                         void* out_last, const ps_table* t, int32_t tsteps, void* stream);

/* ps_two_step_tb restricted to output rows [row_lo, row_hi) of a row slab (boundary rows
 * first, halo exchange, interior concurrently).  A slab needs ghost >= R*tsteps rows
 * holding the neighbours' last R*tsteps rows of u^k and R*(tsteps-1) rows of u^{k-1}. */
ps_status ps_two_step_tb_rows(const ps_grid* g, const void* uk, const void* ukm1,
                              void* out_prev, void* out_last, const ps_table* t, int32_t tsteps,
                              int64_t row_lo, int64_t row_hi, void* stream);

/* ps_two_step_tb_rows with in-kernel halo delivery (the fused pass +
 * exchange over NVLink peer memory): the CTAs that write out_last rows [0, R*tsteps) and
 * [rows - R*tsteps, rows), and out_prev rows [0, R*(tsteps-1)) and [rows - R*(tsteps-1),
 * rows), also store them into the neighbour slabs' ghost rows — up_prev / up_last (the
 * slab above's out_prev / out_last levels, `up_rows` logical rows) at rows up_rows + r,
 * dn_prev / dn_last (the slab below's) at rows r - rows.  Peer pointers are allocation
 * bases (ps_ipc_open) on devices reachable by peer access; NULL = no neighbour (both of a
 * side or neither).  Dirichlet slabs, ghost >= R*tsteps.  The caller orders the next pass
 * after the neighbours' boundary launches (event / NCCL token). */
ps_status ps_two_step_tb_halo(const ps_grid* g, const void* uk, const void* ukm1,
                              void* out_prev, void* out_last, const ps_table* t, int32_t tsteps,
                              int64_t row_lo, int64_t row_hi, void* up_prev, void* up_last,
                              int64_t up_rows, void* dn_prev, void* dn_last, void* stream);

/* nsteps updates over four rotating levels with temporal blocking depth tsteps (1..6);
 * lvl[*newest] = u^k and lvl[*previous] = u^{k-1} on entry and on return.  nsteps not
 * divisible by tsteps finishes with single steps. */
ps_status ps_march_tb(const ps_grid* g, void* lvl[4], int64_t nsteps, const ps_table* t,
                      int32_t tsteps, int32_t* newest, int32_t* previous, void* stream);

/* Tile-resident march for SMALL f64 grids, Dirichlet or periodic (a level of a few MB: BASELINE
 * config 1, the reference's own regime — run()'s loop of two_step calls, simulator.py:
 * 271-274).  One cooperative launch runs all nsteps updates: the grid is cut into one tile
 * per SM, every pass loads a tile plus a halo of R*tsteps points into shared memory, runs
 * tsteps updates there and publishes its tile to the other pair of levels; tiles wait only
 * for their 8 neighbours (release/acquire epoch flags), not for a launch boundary.  Same
 * level bookkeeping as ps_march_tb (four levels; *newest / *previous updated), same bits
 * as nsteps ps_two_step calls.  tsteps 1..16.  Returns PS_ERR_ARG when the grid does not
 * qualify (f32, row slab, Dirichlet ring narrower than the stencil, or no tiling that fits
 * the SMs' shared memory): ps_tile_supported() asks first. */
int32_t ps_tile_supported(const ps_grid* g, const ps_table* t, int32_t tsteps);
ps_status ps_march_tile(const ps_grid* g, void* lvl[4], int64_t nsteps, const ps_table* t,
                        int32_t tsteps, int32_t* newest, int32_t* previous, void* stream);

/* Host-to-host solve with the PCIe copies overlapped: the field part
 * of run() (simulator.py:253-282: u0/v0 in, first step, n_t - 1 two-step updates, the
 * final level out; dump_grid_csv's input), from HOST arrays to a HOST array.
 *
 * Dirichlet grids are cut into row bands marched as a skewed wavefront: band b uploads
 * its rows of u0/v0, advances every one of its rows through all nsteps levels and
 * downloads the finished rows while later bands are still uploading or computing, so
 * the host<->device copies hide behind the stencil work.  Launch j of band b updates
 * rows [S_b - s(j+1), S_{b+1} - s(j+1)) with a skew s = R*tsteps per launch: every row
 * it reads above the band was finished for that level by band b-1's launch j-1 and is
 * not overwritten before band b reads it (ps_solve_plan lists the launches and their
 * ordering; tests/test_host.py checks the plan for races and replays it on the oracle).
 * Per-point arithmetic is unchanged, so out equals ps_first_step + ps_march[_tb] bit
 * for bit.  Periodic grids (rows wrap) run the same sequence unbanded.
 *
 * lvl: four device levels of *g (scratch; contents on return unspecified).  u0_host,
 * v0_host (NULL = zero velocity), out_host: HOST arrays of (rows + a) x (cols + a)
 * elements with row stride host_pitch, a = 1 for periodic grids (the reference's
 * alias row/column), 0 for Dirichlet; pinned memory for full copy bandwidth.
 * nsteps >= 1 = the time level returned (1 = the first step only).  tsteps: temporal
 * blocking depth (1..6; reduced to 1 for tables without a fused kernel at that depth).
 * nbands: 0 = auto (about 1024 rows per band).  Returns when the work is enqueued on
 * `stream`; out_host is valid after the stream synchronises. */
typedef enum ps_solve_kind {
  PS_OP_LOAD = 0,   /* host u0 rows -> level dst0, v0 rows -> level dst1 (zeros if NULL) */
  PS_OP_FIRST = 1,  /* first step: src0 = u0, src1 = v0 -> dst1 = u1                      */
  PS_OP_STEP = 2,   /* two-step: src0 = u^k, src1 = u^{k-1} -> dst1 = u^{k+1}              */
  PS_OP_PASS = 3,   /* fused pass: src0 = u^k, src1 = u^{k-1} -> dst0 = u^{k+T-1}, dst1 = u^{k+T} */
  PS_OP_STORE = 4   /* level src0 rows -> host out                                         */
} ps_solve_kind;
typedef struct ps_solve_op {
  int32_t kind;         /* ps_solve_kind                                                  */
  int32_t band;
  int32_t tsteps;       /* updates the op advances (PASS: T; FIRST/STEP: 1; else 0)       */
  int32_t stream;       /* 0 = upload, 1..nstreams = compute, nstreams + 1 = download     */
  int32_t src0, src1, dst0, dst1;  /* level indices 0..3, -1 = unused                      */
  int64_t row_lo, row_hi;          /* logical rows written (LOAD/STEP/...) or read (STORE) */
  int64_t after0, after1;          /* ops this one waits for besides its stream's order   */
} ps_solve_op;
/* The launch plan ps_solve_host executes (host-only; no GPU needed).  Writes up to
 * max_ops ops and returns how many the plan has (call with ops = NULL to size it), or
 * -ps_status on bad arguments.  radius = the largest stencil radius of the tables. */
int64_t ps_solve_plan(int64_t rows, int32_t radius, int64_t nsteps, int32_t tsteps,
                      int32_t nbands, int32_t nstreams, ps_solve_op* ops, int64_t max_ops);
ps_status ps_solve_host(const ps_grid* g, void* lvl[4], const void* u0_host,
                        const void* v0_host, void* out_host, int64_t host_pitch,
                        const ps_table* tu, const ps_table* tv, const ps_table* t, double tau,
                        int64_t nsteps, int32_t tsteps, int32_t nbands, void* stream);

/* Sum of K isotropic Gaussians sampled at x1 = i/n, x2 = j/n (the reference's node
 * coordinates np.arange(n+1)/n, simulator.py:254-255) in f64, k order:
 *   u = sum_k amp[k] * exp(-((x1-cx[k])^2 + (x2-cy[k])^2) / (2*(width[k]^2)))
 * written in the level's dtype (BASELINE configs 3-5 initial data; the reference's
 * _sample, simulator.py:141-144, evaluates user callables on the same nodes).
 * Dirichlet: the whole (n+1)^2 block incl. ring; periodic: the core, then its images.
 * The parameter arrays are HOST pointers (copied into the launch, K <= 512). */
ps_status ps_gaussian_sum(const ps_grid* g, void* level, int32_t K, const double* cx,
                          const double* cy, const double* width, const double* amp,
                          int64_t n, void* stream);

/* Fused per-step error sums of run() for the standing-wave benchmark (
 * replaces simulator.py:275-280 when `exact` is the default standing wave):
 *   ref = S * st;  out2[0] = sum((u - ref)^2);  out2[1] = sum(ref^2)
 * over the rows_h x cols_h block from logical (0,0) (the reference's (n+1)^2 array incl.
 * ring / alias), summed in numpy's pairwise order so both floats equal the reference's
 * bit for bit.  S (same layout as the level) holds sin(2πx1)*sin(2πx2) as numpy computes
 * it; st = sin(2√2 π c t).  out2 is a DEVICE pointer.  f64 grids only.
 * ps_errsum_create allocates the per-size summation plan (not a hot call). */
typedef struct ps_errsum ps_errsum;
ps_errsum* ps_errsum_create(int64_t rows_h, int64_t cols_h);
ps_status ps_errsum_step(ps_errsum* e, const ps_grid* g, const void* level, const void* S,
                         double st, double* out2, void* stream);
void ps_errsum_destroy(ps_errsum* e);

/* run()'s time loop with the fused metric (simulator.py:271-280): nsteps two-step
 * updates (as ps_march), each followed by ps_errsum_step with st_host[k] (HOST array of
 * nsteps sine factors) into out_dev[2k..2k+1] (DEVICE).  One call, no per-step host sync. */
ps_status ps_march_errsum(const ps_grid* g, void* lvl[3], int64_t nsteps, const ps_table* t,
                          ps_errsum* e, const void* S, const double* st_host, double* out_dev,
                          int32_t* newest, void* stream);

/* Snapshot writer: one HOST rows x cols block as CSV, "%.17g" per
 * value, "," between values, "\n" after each row — the text of the reference's
 * dump_grid_csv (simulator.py:293-295, np.savetxt) byte for byte, without Python
 * formatting cost.  Host-only; pair with an asynchronous ps_copy_out into pinned memory. */
ps_status ps_write_csv(const char* path, const void* host, int64_t rows, int64_t cols,
                       int64_t host_pitch, int32_t dtype);

/* Batched tiny-grid runs: many complete run()s of the paper's tables
 * (reference benchmarks.py:68-95) in one launch, one CTA per simulation with its three
 * levels in shared memory (n <= PS_BATCH_MAX_N).  For each simulation the caller packs a
 * ps_batch_sim into an opaque device descriptor (ps_batch_pack, ps_batch_desc_bytes per
 * descriptor; copy the array to the device) and concatenates, at the given offsets, the
 * (n+1)^2 reference-layout arrays u0, v0 (periodic: alias edges consistent) and
 * S = sin(2πx1)*sin(2πx2), the n_t sine factors st[k-1] = sin(2√2 π c kτ), and room for
 * 2*n_t outputs.  out receives, per step k, sum((u^k - S*st)^2) and sum((S*st)^2) in
 * numpy's pairwise order — run()'s per-step error sums, bit for bit. */
#define PS_BATCH_MAX_N 90
typedef struct ps_batch_sim {
  int32_t n, n_t, bc, pad;
  double tau;
  ps_table first_u, first_v, two_step;
  int64_t off_field, off_st, off_out;
} ps_batch_sim;
size_t ps_batch_desc_bytes(void);
ps_status ps_batch_pack(const ps_batch_sim* sim, void* desc_host);
ps_status ps_batch_run(int32_t nsim, int32_t max_n, const void* desc_dev, const double* u0,
                       const double* v0, const double* S, const double* st, double* out,
                       void* stream);

/* Kernel launches issued by this library since load (for launch accounting). */
int64_t ps_launch_count(void);

/* Static description of a ps_status. */
const char* ps_strerror(int32_t status);

/* Library version string ("paper_1904_04048_b200 <semver> sm_100a"). */
const char* ps_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PS_H_ */
