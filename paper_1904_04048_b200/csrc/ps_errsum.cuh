// ps_errsum.cuh — fused per-step error sums of run().
// Included inside namespace ps by ps_device.cu.
//
// The reference scores every step against the standing wave (simulator.py:275-280):
//     ref      = sin(2π x1) * sin(2π x2) * sin(2√2 π c t)     (= S * st, S fixed)
//     step_num = float(((u - ref) ** 2).sum())
//     step_den = float((ref ** 2).sum())
// numpy's float64 sum over a contiguous array is a pairwise sum with a fixed shape
// (blocks of <= 128 summed with 8 interleaved accumulators, larger ranges split at
// n/2 rounded down to a multiple of 8; ranges < 8 summed sequentially from 0.0).
// The host builds that tree once per size (ps_errsum_create); each step one kernel sums
// the leaves and one single-block kernel folds the tree level by level, so the device
// result is the reference's float bit for bit (checked against golden per-step errors).

struct ErrsumPlan {
  int64_t rows_h = 0, cols_h = 0, count = 0;
  int32_t nleaves = 0, ninternal = 0, nlevels = 0;
  // device arrays
  int64_t* leaf_start = nullptr;
  int32_t* leaf_len = nullptr;
  int32_t* node_left = nullptr;   // per internal node (level-sorted), child ids
  int32_t* node_right = nullptr;
  int32_t* node_id = nullptr;     // value slot of each internal node
  int32_t* level_off = nullptr;   // [nlevels + 1]
  double* values = nullptr;       // [2 * (nleaves + ninternal)] : num | den
  int32_t root = 0;
  std::vector<int32_t> h_level_off;
};

constexpr int kPwBlock = 128;  // numpy PW_BLOCKSIZE

__device__ __forceinline__ void errsum_terms(const double* u, const double* S, int64_t pitch,
                                             int64_t cols_h, int64_t f, double st, double& d2,
                                             double& r2) {
  const int64_t i = f / cols_h;
  const int64_t j = f - i * cols_h;
  const double ref = __dmul_rn(S[i * pitch + j], st);
  const double d = __dsub_rn(u[i * pitch + j], ref);
  d2 = __dmul_rn(d, d);
  r2 = __dmul_rn(ref, ref);
}

// One leaf per 8 lanes: lane j runs numpy's j-th interleaved accumulator (elements
// j, j+8, j+16, ... of the leaf's multiple-of-8 part), the 8 partial sums combine by
// shuffle in numpy's fixed order ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), and lane 0 adds the
// tail sequentially.  Leaves shorter than 8 are summed sequentially from 0.0 by lane 0.
__global__ void __launch_bounds__(256)
    k_errsum_leaves(const double* __restrict__ u, const double* __restrict__ S, int64_t pitch,
                    int64_t cols_h, double st, const int64_t* __restrict__ leaf_start,
                    const int32_t* __restrict__ leaf_len, int32_t nleaves,
                    double* __restrict__ values, int32_t nvalues) {
  const int64_t gt = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int leaf = int(gt >> 3), j = int(gt & 7);
  const bool valid = leaf < nleaves;
  int64_t a = 0;
  int n = 0;
  if (valid) {
    a = leaf_start[leaf];
    n = leaf_len[leaf];
  }
  const int full = n - (n % 8);
  double rn = 0.0, rd = 0.0;
  if (n >= 8) {
    errsum_terms(u, S, pitch, cols_h, a + j, st, rn, rd);
    for (int x = 8 + j; x < full; x += 8) {
      double d2, r2;
      errsum_terms(u, S, pitch, cols_h, a + x, st, d2, r2);
      rn = __dadd_rn(rn, d2);
      rd = __dadd_rn(rd, r2);
    }
  }
  // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) across the leaf's 8 lanes
#pragma unroll
  for (int w = 1; w < 8; w <<= 1) {
    const double on = __shfl_down_sync(0xffffffffu, rn, w, 8);
    const double od = __shfl_down_sync(0xffffffffu, rd, w, 8);
    rn = __dadd_rn(rn, on);
    rd = __dadd_rn(rd, od);
  }
  if (!valid || j != 0) return;
  double num, den;
  int x;
  if (n < 8) {
    num = 0.0;
    den = 0.0;
    x = 0;
  } else {
    num = rn;
    den = rd;
    x = full;
  }
  for (; x < n; ++x) {
    double d2, r2;
    errsum_terms(u, S, pitch, cols_h, a + x, st, d2, r2);
    num = __dadd_rn(num, d2);
    den = __dadd_rn(den, r2);
  }
  values[leaf] = num;
  values[nvalues + leaf] = den;
}

__global__ void __launch_bounds__(1024)
    k_errsum_fold(const int32_t* __restrict__ node_left, const int32_t* __restrict__ node_right,
                  const int32_t* __restrict__ node_id, const int32_t* __restrict__ level_off,
                  int32_t nlevels, double* __restrict__ values, int32_t nvalues, int32_t root,
                  double* __restrict__ out2) {
  for (int lv = 0; lv < nlevels; ++lv) {
    for (int k = level_off[lv] + threadIdx.x; k < level_off[lv + 1]; k += blockDim.x) {
      const int id = node_id[k], l = node_left[k], r = node_right[k];
      values[id] = __dadd_rn(values[l], values[r]);
      values[nvalues + id] = __dadd_rn(values[nvalues + l], values[nvalues + r]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out2[0] = values[root];
    out2[1] = values[nvalues + root];
  }
}
