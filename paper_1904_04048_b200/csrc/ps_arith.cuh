// ps_arith.cuh — per-point arithmetic contracts (see ps_arith in include/ps.h).
//
// The reference accumulates each stencil as  acc = zeros(); acc += coeff * shifted
// (simulator.py:152-160): a +0.0 start, one rounded product and one rounded add per
// tap, in table order, never fused.  Every operation below is an explicit _rn
// intrinsic so nvcc cannot contract a multiply-add into an FMA.
#pragma once

namespace ps {

enum { ARITH_REF = 0, ARITH_NATIVE = 1 };

template <typename T, int A>
struct Arith;

// f64: the reference's float64 path (both contracts coincide).
template <int A>
struct Arith<double, A> {
  using acc_t = double;
  using coef_t = double;
  __device__ __forceinline__ static acc_t zero() { return 0.0; }
  __device__ __forceinline__ static acc_t tap(acc_t acc, coef_t c, double u) {
    return __dadd_rn(acc, __dmul_rn(c, u));
  }
  // tap() in two halves: the separately rounded product fl(c*u) — the same value for
  // every output point that reads u through a tap with this coefficient, so the fused
  // kernels compute it once per input element and coefficient class — and the add
  static constexpr bool kSplit = true;
  static constexpr bool kPair = false;
  __device__ __forceinline__ static acc_t mul(coef_t c, double u) { return __dmul_rn(c, u); }
  __device__ __forceinline__ static acc_t add(acc_t acc, acc_t p) { return __dadd_rn(acc, p); }
  // u^{k+1} = acc - u^{k-1}            (simulator.py:184)
  __device__ __forceinline__ static double two(acc_t acc, double ukm1) {
    return __dsub_rn(acc, ukm1);
  }
  // u^1 = acc_u + tau * acc_v           (simulator.py:178-179)
  __device__ __forceinline__ static double first(acc_t au, acc_t av, double tau) {
    return __dadd_rn(au, __dmul_rn(tau, av));
  }
  // velocity half of the first step, negated: two(acc_u, vpart(acc_v)) == first(acc_u,
  // acc_v) bit for bit, because a - (-b) = a + b exactly in IEEE arithmetic
  __device__ __forceinline__ static double vpart(acc_t av, double tau) {
    return -__dmul_rn(tau, av);
  }
};

// f32, reference contract: numpy multiplies a float32 field by a Python float in
// float32, adds the product into the float64 accumulator, stores the accumulator
// back into a float32 array and subtracts in float32 (simulator.py:150-154, 184).
template <>
struct Arith<float, ARITH_REF> {
  using acc_t = double;
  using coef_t = float;
  __device__ __forceinline__ static acc_t zero() { return 0.0; }
  __device__ __forceinline__ static acc_t tap(acc_t acc, coef_t c, float u) {
    return __dadd_rn(acc, static_cast<double>(__fmul_rn(c, u)));
  }
  static constexpr bool kPair = false;
  static constexpr bool kSplit = true;   // product = the f32 product widened once
  __device__ __forceinline__ static acc_t mul(coef_t c, float u) {
    return static_cast<double>(__fmul_rn(c, u));
  }
  __device__ __forceinline__ static acc_t add(acc_t acc, acc_t p) { return __dadd_rn(acc, p); }
  __device__ __forceinline__ static float two(acc_t acc, float ukm1) {
    return __fsub_rn(__double2float_rn(acc), ukm1);
  }
  __device__ __forceinline__ static float first(acc_t au, acc_t av, float tau) {
    return __fadd_rn(__double2float_rn(au), __fmul_rn(tau, __double2float_rn(av)));
  }
  __device__ __forceinline__ static float vpart(acc_t av, float tau) {
    return -__fmul_rn(tau, __double2float_rn(av));
  }
};

// f32, native contract: the taps in the same table order, each folded in with one
// correctly rounded fused multiply-add (acc = fma(c, u, acc) from +0.0), then a float32
// subtract (first step: acc_u + fl(tau * acc_v)).  Half the floating-point instructions of the reference sequence and at
// least as accurate; checked bit for bit against the oracle's fmaf() chain and against
// the f64 run within the stated tolerance.
template <>
struct Arith<float, ARITH_NATIVE> {
  using acc_t = float;
  using coef_t = float;
  __device__ __forceinline__ static acc_t zero() { return 0.0f; }
  __device__ __forceinline__ static acc_t tap(acc_t acc, coef_t c, float u) {
    return __fmaf_rn(c, u, acc);
  }
  static constexpr bool kSplit = false;  // one fused operation per tap: nothing to share
  // Two taps of neighbouring outputs in one instruction: sm_100's packed fma.rn.f32x2 (SASS
  // FFMA2) performs two independent correctly rounded FMAs on a register pair, with the
  // coefficient broadcast to both halves — the same bits as two tap() calls for half the
  // issue slots (the fused f32 kernels are issue-bound, not FMA-pipe-bound).
  static constexpr bool kPair = true;
  __device__ __forceinline__ static void tap2(acc_t& a0, acc_t& a1, coef_t c, float u0,
                                              float u1) {
    uint64_t ra, ru, rc;
    asm("mov.b64 %0, {%1, %2};" : "=l"(ra) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(ru) : "f"(u0), "f"(u1));
    asm("mov.b64 %0, {%1, %1};" : "=l"(rc) : "f"(c));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(ra) : "l"(rc), "l"(ru));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(ra));
  }
  __device__ __forceinline__ static float two(acc_t acc, float ukm1) {
    return __fsub_rn(acc, ukm1);
  }
  // two() for a pair of outputs: packed sub.rn.f32x2, the same two rounded subtractions
  __device__ __forceinline__ static void two2(float& r0, float& r1, acc_t a0, acc_t a1,
                                              float m0, float m1) {
    uint64_t ra, rm, rr;
    asm("mov.b64 %0, {%1, %2};" : "=l"(ra) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(rm) : "f"(m0), "f"(m1));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(rr) : "l"(ra), "l"(rm));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r0), "=f"(r1) : "l"(rr));
  }
  // first step: acc_u + fl(tau * acc_v) (unfused, so it decomposes like the others)
  __device__ __forceinline__ static float first(acc_t au, acc_t av, float tau) {
    return __fadd_rn(au, __fmul_rn(tau, av));
  }
  __device__ __forceinline__ static float vpart(acc_t av, float tau) {
    return -__fmul_rn(tau, av);
  }
};

}  // namespace ps
