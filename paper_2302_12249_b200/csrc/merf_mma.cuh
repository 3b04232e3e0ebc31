// merf_mma.cuh -- warp-level mma.sync building blocks of the deferred MLP (Eq. 3):
// split-fp16 operand pairs, m16n8k16 / m16n8k8 products, ldmatrix staging.  Shared by the
// shade kernel (merf_shade_mma.cu) and the march kernel's fused epilogue (KF_FUSED).
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

namespace merf {

constexpr int kXStride = 56;   // halves per staged input row (48 used; 112 B rows: ldmatrix conflict-free)

__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

// (a, b) -> packed fp16 hi pair and the fp16 pair of the residuals
__device__ __forceinline__ void split2(float a, float b, uint32_t& hi, uint32_t& lo) {
    const __half2 h = __floats2half2_rn(a, b);
    const float2 hf = __half22float2(h);
    hi = h2u(h);
    lo = h2u(__floats2half2_rn(a - hf.x, b - hf.y));
}

__device__ __forceinline__ float wnk(const float* w, int off, int nin, int nout, int n, int k) {
    return (n < nout && k < nin) ? w[off + n * nin + k] : 0.f;
}

__device__ __forceinline__ void mma16(float c[4], const uint32_t a[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma8(float c[4], uint32_t a0, uint32_t a1, uint32_t b0) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a0), "r"(a1), "r"(b0));
}
__device__ __forceinline__ void ldm4(uint32_t a[4], const void* p) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(p);
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]) : "r"(s));
}
__device__ __forceinline__ void ldm2(uint32_t& a0, uint32_t& a1, const void* p) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(p);
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(a0), "=r"(a1) : "r"(s));
}

// hi/lo x (hi, lo) products of one m16n8 tile: c += A_hi B_hi + A_hi B_lo + A_lo B_hi
__device__ __forceinline__ void mma16x3(float c[4], const uint32_t ah[4], const uint32_t al[4], const uint32_t* b) {
    mma16(c, al, b[0], b[1]);
    mma16(c, ah, b[2], b[3]);
    mma16(c, ah, b[0], b[1]);
}

// ReLU of two n8 accumulator tiles of one m16 tile -> the hi/lo A fragments of the next layer
// (C of n tiles 0/1 at rows g, g+8 == A columns 2t.. / 2t+8.. at rows g, g+8)
__device__ __forceinline__ void relu_to_a(const float c0[4], const float c1[4], uint32_t ah[4], uint32_t al[4]) {
    split2(fmaxf(c0[0], 0.f), fmaxf(c0[1], 0.f), ah[0], al[0]);
    split2(fmaxf(c0[2], 0.f), fmaxf(c0[3], 0.f), ah[1], al[1]);
    split2(fmaxf(c1[0], 0.f), fmaxf(c1[1], 0.f), ah[2], al[2]);
    split2(fmaxf(c1[2], 0.f), fmaxf(c1[3], 0.f), ah[3], al[3]);
}


}  // namespace merf
