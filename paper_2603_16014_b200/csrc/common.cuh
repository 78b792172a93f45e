// Shared device helpers for the fastmtgp-b200 kernels (sm_100a, fp64).
#pragma once

#include <utility>

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

namespace fmtgp {

constexpr int MAXD = 16;   // spatial dimensions supported by the register-resident kernels
constexpr int MAXT = 8;    // tasks (reference make_design: L <= 8, ld_sequences.cpp:167)
constexpr int MAXP = MAXT * (MAXT + 1) / 2;
constexpr int DIGITAL_BITS = 53;
constexpr uint64_t MASK53 = (uint64_t(1) << 53) - 1;
constexpr int TW_BASE_LOG = 13;  // twiddle tables hold 2^13 entries per level

// ---------------------------------------------------------------- complex fp64
__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__host__ __device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
    return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__host__ __device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__host__ __device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }

// ---------------------------------------------------------------- twiddles
// tw[L][u] = exp(-2 pi i u / 2^L) for u < min(2^L, 2^13), L = 0..26, built on device
// with sincospi (see transforms.cu).  exp(-2 pi i t / 2^L) for any t < 2^L is one
// table read (L <= 13) or the product of two (L > 13): t = hi * 2^(L-13) + lo.
struct Twiddles {
    const double2* tab;  // [27][8192]
};

__device__ __forceinline__ double2 twiddle(const double2* __restrict__ tab, uint64_t t, int L) {
    // exp(-2 pi i t / 2^L), t taken mod 2^L
    t &= (uint64_t(1) << L) - 1;
    if (L <= TW_BASE_LOG) return __ldg(tab + (size_t(L) << TW_BASE_LOG) + t);
    const int s = L - TW_BASE_LOG;
    const double2 hi = __ldg(tab + (size_t(TW_BASE_LOG) << TW_BASE_LOG) + (t >> s));
    const double2 lo = __ldg(tab + (size_t(L) << TW_BASE_LOG) + (t & ((uint64_t(1) << s) - 1)));
    return cmul(hi, lo);
}

// ---------------------------------------------------------------- async global -> shared copies (LDGSTS)
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
// One element of a global -> shared staging loop (double or double2), issued asynchronously so a
// thread keeps all of its loads in flight; pair with cp_async_wait_all() before the barrier.
template <class T>
__device__ __forceinline__ void cp_async_el(T* smem, const T* gmem) {
    static_assert(sizeof(T) == 8 || sizeof(T) == 16, "cp_async_el: 8 or 16 bytes");
    if constexpr (sizeof(T) == 16) cp_async16(smem, gmem);
    else cp_async8(smem, gmem);
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// ---------------------------------------------------------------- programmatic dependent launch
// A kernel launched with launch_pdl() may start while its predecessor in the stream is still
// running; it runs its independent prologue (prefetches) and then pdl_wait()s, which returns once
// the predecessor grid has completed and its writes are visible.  pdl_trigger() lets the
// dependent grid be scheduled early (safe anywhere: the dependent still pdl_wait()s).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// a failing launch also sets the runtime's last error, which the caller's cudaGetLastError() check reads
#define CK_LAUNCH(x) ((void)(x))

template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                              Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------- reductions
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* scratch /* >= NT/32 */) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) scratch[w] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x < 32) {
        r = (l < NT / 32) ? scratch[l] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    }
    return r;  // valid in thread 0
}

// K block sums with a single barrier pair: warp shuffles, one smem transpose, warp 0 folds.
// scratch >= (NT/32) * K doubles; results valid in thread 0 (out[k]).
template <int NT, int K>
__device__ __forceinline__ void block_sum_vec(double (&v)[K], double* scratch) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < K; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    }
    __syncthreads();
    if (l == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) scratch[w * K + k] = v[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double s = 0.0;
            for (int ww = 0; ww < NT / 32; ++ww) s += scratch[ww * K + k];
            v[k] = s;
        }
    }
}

// double(t) for t < 2^32 without I2F.F64: that conversion issues at a quarter of the DFMA rate on
// B200 (profiles/r02_fp64_peak.log: 4.4 Tconv/s vs 17 T DFMA/s); 2^52 + t is t in the low
// mantissa bits of a constant exponent (an integer move), one exact DADD removes the 2^52
__device__ __forceinline__ double u32_to_f64(uint32_t t) { return __hiloint2double(0x43300000, int(t)) - 0x1p52; }

__device__ __forceinline__ uint32_t bitrev32(uint32_t x, int m) { return m == 0 ? 0u : (__brev(x) >> (32 - m)); }
__device__ __forceinline__ uint64_t bitrev64(uint64_t x, int m) { return m == 0 ? 0ull : (__brevll(x) >> (64 - m)); }

// ---------------------------------------------------------------- real / complex scalar ops
template <bool CX>
struct Sc;
template <>
struct Sc<true> {
    using T = double2;
    static __device__ __forceinline__ T zero() { return make_double2(0.0, 0.0); }
    static __device__ __forceinline__ T one() { return make_double2(1.0, 0.0); }
    static __device__ __forceinline__ T add(T a, T b) { return cadd(a, b); }
    static __device__ __forceinline__ T mul(T a, T b) { return cmul(a, b); }
    static __device__ __forceinline__ T mulc(T a, T b) { return cmulc(a, b); }  // a conj(b)
    static __device__ __forceinline__ T conj(T a) { return cconj(a); }
    static __device__ __forceinline__ T sub(T a, T b) { return csub(a, b); }
    static __device__ __forceinline__ T scale(T a, double s) { return cscale(a, s); }
    static __device__ __forceinline__ double re(T a) { return a.x; }
    static __device__ __forceinline__ double im(T a) { return a.y; }
    static __device__ __forceinline__ double abs2(T a) { return a.x * a.x + a.y * a.y; }
};
template <>
struct Sc<false> {
    using T = double;
    static __device__ __forceinline__ T zero() { return 0.0; }
    static __device__ __forceinline__ T one() { return 1.0; }
    static __device__ __forceinline__ T add(T a, T b) { return a + b; }
    static __device__ __forceinline__ T mul(T a, T b) { return a * b; }
    static __device__ __forceinline__ T mulc(T a, T b) { return a * b; }
    static __device__ __forceinline__ T conj(T a) { return a; }
    static __device__ __forceinline__ T sub(T a, T b) { return a - b; }
    static __device__ __forceinline__ T scale(T a, double s) { return a * s; }
    static __device__ __forceinline__ double re(T a) { return a; }
    static __device__ __forceinline__ double im(T) { return 0.0; }
    static __device__ __forceinline__ double abs2(T a) { return a * a; }
};

}  // namespace fmtgp
