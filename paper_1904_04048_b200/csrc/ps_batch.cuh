// ps_batch.cuh — batched tiny-grid runs.  Included inside namespace ps
// by ps_device.cu.
//
// The paper's accuracy tables (reference benchmarks.py:27-61) are dozens of run() calls
// on grids of at most 81^2 nodes.  One CTA per simulation keeps its three levels in
// shared memory (<= ~200 KB) and runs the whole simulation — first step, n_t - 1
// two-step updates, and after every step the reference's error sums in numpy's
// pairwise order (simulator.py:275-280) — so a whole table is one kernel launch.
// Per-point arithmetic is Arith<double, REF> with runtime tap tables in dict order;
// results equal run()'s bit for bit.
//
// Periodic levels store the reference's (n+1)^2 array; the core is updated with wrap
// indexing and the alias row/column is copied from the core afterwards, which is what
// run() produces (its u^{k-1} alias is always consistent, simulator.py:258-260).

constexpr int kBatchThreads = 512;
constexpr int kBatchMaxLeaves = 256;

struct BatchTable {
  int32_t n;
  int8_t q1[PS_MAX_TAPS], q2[PS_MAX_TAPS];
  double c[PS_MAX_TAPS];
};

__device__ __forceinline__ double batch_acc(const BatchTable& t, const double* L, int N1, int n,
                                            bool per, int i, int j) {
  double acc = 0.0;
  for (int s = 0; s < t.n; ++s) {
    int ii = i + t.q1[s], jj = j + t.q2[s];
    if (per) {
      ii %= n;
      ii += ii < 0 ? n : 0;
      jj %= n;
      jj += jj < 0 ? n : 0;
    }
    acc = __dadd_rn(acc, __dmul_rn(t.c[s], L[ii * N1 + jj]));
  }
  return acc;
}

struct BatchDev {
  int32_t n, nt, bc;
  double tau;
  BatchTable tu, tv, t2;
  int64_t off_field, off_st, off_out;
};

// numpy pairwise-sum leaves of a length-N range (<= kBatchMaxLeaves), built by thread 0
// with an explicit stack; internal nodes come out in post-order (children first).
__device__ void batch_build_tree(int N, int* leaf_start, int* leaf_len, int* nleaves,
                                 int* node_l, int* node_r, int* nnodes) {
  struct Fr {
    int start, n, state, left;
  };
  Fr st[32];
  int sp = 0, ret = 0, nl = 0, nn = 0;
  st[sp++] = {0, N, 0, 0};
  while (sp) {
    Fr& f = st[sp - 1];
    if (f.n <= 128) {
      leaf_start[nl] = f.start;
      leaf_len[nl] = f.n;
      ret = nl++;  // leaves are ids [0, kBatchMaxLeaves)
      --sp;
      continue;
    }
    int n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.state == 0) {
      f.state = 1;
      st[sp++] = {f.start, n2, 0, 0};
    } else if (f.state == 1) {
      f.state = 2;
      f.left = ret;
      st[sp++] = {f.start + n2, f.n - n2, 0, 0};
    } else {
      node_l[nn] = f.left;
      node_r[nn] = ret;
      ret = kBatchMaxLeaves + nn++;  // internal ids follow the leaves
      --sp;
    }
  }
  *nleaves = nl;
  *nnodes = nn;
}

__global__ void __launch_bounds__(kBatchThreads)
    k_batch_run(const BatchDev* __restrict__ sims, const double* __restrict__ u0s,
                const double* __restrict__ v0s, const double* __restrict__ Ss,
                const double* __restrict__ sts, double* __restrict__ outs) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const BatchDev& sim = sims[blockIdx.x];
  const int n = sim.n, N1 = n + 1, NN = N1 * N1;
  const bool per = sim.bc == PS_BC_PERIODIC;
  double* L0 = reinterpret_cast<double*>(smem_raw);
  double* lv[3] = {L0, L0 + NN, L0 + 2 * NN};
  double* vals = L0 + 3 * NN;                          // 2 * (leaves + nodes)
  int* leaf_start = reinterpret_cast<int*>(vals + 4 * kBatchMaxLeaves);
  int* leaf_len = leaf_start + kBatchMaxLeaves;
  int* node_l = leaf_len + kBatchMaxLeaves;
  int* node_r = node_l + kBatchMaxLeaves;
  int* counts = node_r + kBatchMaxLeaves;              // nleaves, nnodes
  const double* u0 = u0s + sim.off_field;
  const double* v0 = v0s + sim.off_field;
  const double* S = Ss + sim.off_field;
  const double* stv = sts + sim.off_st;
  double* out = outs + sim.off_out;
  const int tid = threadIdx.x;

  if (tid == 0) batch_build_tree(NN, leaf_start, leaf_len, &counts[0], node_l, node_r, &counts[1]);
  for (int p = tid; p < NN; p += blockDim.x) {
    lv[1][p] = u0[p];  // u^0
    lv[0][p] = v0[p];  // v0 (its level is recycled after the first step)
  }
  __syncthreads();

  auto alias = [&](double* L) {  // periodic: copy the core onto row/col n (_alias_edges)
    __syncthreads();
    for (int i = tid; i < n; i += blockDim.x) L[i * N1 + n] = L[i * N1];
    __syncthreads();
    for (int j = tid; j < N1; j += blockDim.x) L[n * N1 + j] = L[j];
    __syncthreads();
  };

  auto errsum = [&](const double* L, int k) {  // step k (1-based) into out[2k-2 .. 2k-1]
    const double st = stv[k - 1];
    const int nl = counts[0], nn = counts[1];
    // 8 lanes per leaf; every lane of a warp runs the same number of rounds so the
    // width-8 shuffles below always see full warps
    for (int base = 0; base < nl * 8; base += blockDim.x) {
      const int w = base + tid;
      const bool on = w < nl * 8;
      const int leaf = on ? (w >> 3) : 0, j = w & 7;
      const int a = on ? leaf_start[leaf] : 0, len = on ? leaf_len[leaf] : 0;
      const int full = len - (len % 8);
      auto term = [&](int f, double& d2, double& r2) {
        const double ref = __dmul_rn(S[f], st);
        const double d = __dsub_rn(L[f], ref);
        d2 = __dmul_rn(d, d);
        r2 = __dmul_rn(ref, ref);
      };
      double rn = 0.0, rd = 0.0;
      if (len >= 8) {
        term(a + j, rn, rd);
        for (int x = 8 + j; x < full; x += 8) {
          double d2, r2;
          term(a + x, d2, r2);
          rn = __dadd_rn(rn, d2);
          rd = __dadd_rn(rd, r2);
        }
      }
      // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) across the leaf's 8 lanes
#pragma unroll
      for (int off = 1; off < 8; off <<= 1) {
        const double xn = __shfl_down_sync(0xffffffffu, rn, off, 8);
        const double xd = __shfl_down_sync(0xffffffffu, rd, off, 8);
        rn = __dadd_rn(rn, xn);
        rd = __dadd_rn(rd, xd);
      }
      if (on && j == 0) {
        double num, den;
        int x;
        if (len < 8) {
          num = den = 0.0;
          x = 0;
        } else {
          num = rn;
          den = rd;
          x = full;
        }
        for (; x < len; ++x) {
          double d2, r2;
          term(a + x, d2, r2);
          num = __dadd_rn(num, d2);
          den = __dadd_rn(den, r2);
        }
        vals[leaf] = num;
        vals[kBatchMaxLeaves + leaf] = den;
      }
    }
    __syncthreads();
    if (tid == 0) {
      // internal nodes in post-order; their values live after the leaves'
      double* nv = vals + 2 * kBatchMaxLeaves;
      auto get = [&](int id, int half) {
        return id < kBatchMaxLeaves ? vals[half * kBatchMaxLeaves + id]
                                    : nv[2 * (id - kBatchMaxLeaves) + half];
      };
      double rn = vals[0], rd = vals[kBatchMaxLeaves];
      for (int m = 0; m < nn; ++m) {
        rn = __dadd_rn(get(node_l[m], 0), get(node_r[m], 0));
        rd = __dadd_rn(get(node_l[m], 1), get(node_r[m], 1));
        nv[2 * m] = rn;
        nv[2 * m + 1] = rd;
      }
      out[2 * (k - 1)] = rn;
      out[2 * (k - 1) + 1] = rd;
    }
    __syncthreads();
  };

  // ---- first step: u^1 into lv[2] (simulator.py:178-179, 269-270)
  for (int p = tid; p < NN; p += blockDim.x) {
    const int i = p / N1, j = p - i * N1;
    double v = 0.0;
    if (per ? (i < n && j < n) : (i >= 1 && i < n && j >= 1 && j < n)) {
      const double au = batch_acc(sim.tu, lv[1], N1, n, per, i, j);
      const double av = batch_acc(sim.tv, lv[0], N1, n, per, i, j);
      v = __dadd_rn(au, __dmul_rn(sim.tau, av));
    }
    lv[2][p] = v;
  }
  if (per) alias(lv[2]);
  __syncthreads();
  errsum(lv[2], 1);

  // ---- two-step updates (simulator.py:183-191, 273-274)
  int cur = 2, prev = 1;
  for (int k = 2; k <= sim.nt; ++k) {
    const int nxt = 3 - cur - prev;
    for (int p = tid; p < NN; p += blockDim.x) {
      const int i = p / N1, j = p - i * N1;
      double v = 0.0;
      if (per ? (i < n && j < n) : (i >= 1 && i < n && j >= 1 && j < n))
        v = __dsub_rn(batch_acc(sim.t2, lv[cur], N1, n, per, i, j), lv[prev][p]);
      lv[nxt][p] = v;
    }
    if (per) alias(lv[nxt]);
    __syncthreads();
    errsum(lv[nxt], k);
    prev = cur;
    cur = nxt;
  }
}
