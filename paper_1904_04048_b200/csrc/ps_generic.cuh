// ps_generic.cuh — generic (runtime tap list) update, periodic image refresh and
// Gaussian-sum initial data.  Included inside namespace ps by ps_device.cu.
#pragma once

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

