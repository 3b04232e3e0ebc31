// merf_device.cuh -- device-side building blocks of libmerf (sm_100a).
//
// Canonical fp64 ray setup (reading D8 in DESIGN.md): every fp64 operation that decides
// the integer lattice (ray generation, region segmentation, contraction of segment
// endpoints, segment length/direction, llrint to the 2^-28 lattice, F = MERF_FIXED_BITS) uses the _rn
// intrinsics so that nvcc can never contract a multiply-add into an FMA.  The same
// IEEE-754 operations in the same order give bit-identical lattices on any conforming
// implementation (e.g. an fp64 CPU reference), which makes per-ray visited-cell traces
// comparable bit for bit.  Shading after the lattice is fp32.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/merf.h"

namespace merf {

constexpr int kF = MERF_FIXED_BITS;                       // lattice fraction bits (28)
constexpr int64_t kOne = int64_t(1) << kF;                // contracted 1.0
constexpr int64_t kTwo = int64_t(1) << (kF + 1);          // contracted 2.0
constexpr int kTwoI = 1 << (kF + 1);                      // contracted 2.0 (int32 lattice)
constexpr int kMaxSeg = 7;                                // convex regions: <= 7 per ray
// A ray that starts in the core (camera origin with ||o||_inf <= 1) has at most 4 segments: the
// core, then the argmax of |x_i(t)| over t past the core exit.  The exit axis j has |x_j|
// increasing with slope |d_j| from then on; another |x_i| is convex piecewise linear with
// slopes +-|d_i|, so it can overtake only if |d_i| > |d_j|, and once it has it keeps growing
// (x_i is past its zero).  Each switch therefore goes to an axis with a strictly larger |d|:
// at most 3 outer regions.  (Measured: 300k random in-core rays, max 4; rays from outside the
// core reach 5 and up to 7 in principle.)  Chunks whose cameras all start in the core use
// 4 slots per ray (128 B instead of 224 B of segment workspace).
constexpr int kMaxSegCore = 4;
constexpr int kMaxCams = 16;                              // cameras per launch (kernel params)
constexpr int kMlpFloats = 883;
constexpr int kMlpFragWords = 44;                         // per-lane words of the mma MLP table

struct DevScene {
    // appearance layouts, pair-interleaved along the fastest axis: entry (.., u) holds texels u
    // and u+1 as 4 words (c1 c1' c2 c2' | c3 c3' c4 c4' | c5 c5' c6 c6' | c7 c7' c0 c0'), so
    // one 16-byte load feeds 7 dp2a directly (no byte gathering)
    const uint4* plane_pairs;     // [3][R + 1][R]: row R of each plane repeats row R - 1
    const int32_t* block_index;   // [(L/8)^3]
    const uint4* atlas_pairs;     // [n_blocks][9][9][8]
    const uint32_t* occ[MERF_MAX_LEVELS];
    const uint32_t* occ_fin;      // = occ[n_levels - 1] (static offset: no dynamic param indexing)
    int n_fin, s_fin;             // = level_res / level_shift of the finest level
    // per finest cell, the lattice shift of the coarsest EMPTY dyadic cell containing it,
    // minus 16 (one byte per entry, x fastest, over the (N_f + 2)^3 BORDERED grid whose border
    // repeats the clamped edge cells); 0 = occupied.  Derived exactly from the finest level;
    // NULL when that level is too large for it (then the level search runs).
    const uint32_t* skiptab;
    const float* mlp;             // [883]
    // per-lane mma fragments of the MLP (merf_shade_mma.cu); NULL = FFMA shade kernel
    const uint32_t* mlp_frag;     // [32][kMlpFragWords]
    int L, R, nb, n_levels;
    int n_blocks_dev;             // atlas blocks (bounds checks of MERF_BOUNDS_CHECK builds)
    int level_res[MERF_MAX_LEVELS];
    int level_shift[MERF_MAX_LEVELS];   // F + 2 - log2(N)
    int sV, sP;                   // F + 2 - log2(L), F + 2 - log2(R)
    float kd, ka;                 // 2m/255 (density / appearance)
    float md, ma;                 // m (density / appearance)
    float kd_l2, md_l2, log2_step;   // base-2 forms: log2(tau Delta) = s kd_l2 - n md_l2 + log2_step
    float kd_l2w;                 // kd_l2 / 65535 (density sum in 16-bit weight units)
    float ka_l2n, ma_l2;          // sigmoid argument: -x log2e = acc ka_l2n + n ma_l2
    float dens_off4, ma_l2_4;     // the n = 4 constants: fmaf(4, -md_l2, log2_step), 4 ma_l2
    int n_src;                    // active sources (V counted only when L > 0)
    int use_v, use_p[3];
    double step;                  // Delta (power of two)
    double lattice_step;          // Delta * 2^F (exact)
    double inv_step;              // 1 / Delta (exact: Delta is a power of two, validated)
    float step_f, t_min, alpha_skip;
};

// The deferred MLP's weights as a kernel parameter: every thread reads the same weight at the
// same time, so they belong in the constant bank (FFMA with a c[][] operand, no load
// instruction); 3.5 KB of the 32 KB parameter space.
struct MlpParams {
    float w[kMlpFloats];
};

struct CamBatch {
    merf_camera cam[kMaxCams];
    int n;
};

// ------------------------------------------------------------------------------------
// exact fp64 helpers (never fused)
// ------------------------------------------------------------------------------------
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

// region_of: 0 = core iff ||x||_inf <= 1 (D2); else 1 + 2j + (x_j < 0) with j
// the first index of max |x_j| (D1).
__device__ __forceinline__ int region_of(double x0, double x1, double x2) {
    double ax = fabs(x0), ay = fabs(x1), az = fabs(x2);
    double m = ax;
    if (ay > m) m = ay;
    if (az > m) m = az;
    if (m <= 1.0) return 0;
    int j = (ax == m) ? 0 : ((ay == m) ? 1 : 2);
    double xj = (j == 0) ? x0 : ((j == 1) ? x1 : x2);
    return 1 + 2 * j + (xj < 0.0 ? 1 : 0);
}

// contract_pi with region g's formula: c_j = s(2 - 1/|x_j|), c_k = x_k/|x_j|.
__device__ __forceinline__ void contract_region(int g, const double x[3], double c[3]) {
    if (g == 0) { c[0] = x[0]; c[1] = x[1]; c[2] = x[2]; return; }
    int j = (g - 1) >> 1;
    bool neg = ((g - 1) & 1) != 0;
    double a = fabs(j == 0 ? x[0] : (j == 1 ? x[1] : x[2]));   // no dynamic indexing
#pragma unroll
    for (int k = 0; k < 3; k++) {
        if (k == j) {
            double v = sub_rn(2.0, div_rn(1.0, a));
            c[k] = neg ? -v : v;
        } else {
            c[k] = div_rn(x[k], a);
        }
    }
}

// lim_{t->inf} contract_g(o + t d): c_j = 2s, c_k = d_k / |d_j|.
__device__ __forceinline__ void vanishing_point(int g, const double d[3], double c[3]) {
    int j = (g - 1) >> 1;
    bool neg = ((g - 1) & 1) != 0;
    double a = fabs(j == 0 ? d[0] : (j == 1 ? d[1] : d[2]));
#pragma unroll
    for (int k = 0; k < 3; k++) c[k] = (k == j) ? (neg ? -2.0 : 2.0) : div_rn(d[k], a);
}

__device__ __forceinline__ void point_at(const double o[3], const double d[3], double t,
                                         double x[3]) {
#pragma unroll
    for (int k = 0; k < 3; k++) x[k] = add_rn(o[k], mul_rn(t, d[k]));
}

// Pinhole ray through the centre of pixel (i, j) (reading D18).
__device__ __forceinline__ void raygen(const merf_camera& c, int i, int j, double o[3],
                                       double d[3]) {
    double x0 = div_rn(sub_rn(add_rn((double)i, 0.5), c.cx), c.fx);
    double x1 = div_rn(sub_rn(add_rn((double)j, 0.5), c.cy), c.fy);
    double v[3];
#pragma unroll
    for (int r = 0; r < 3; r++) {
        double s = add_rn(mul_rn(c.c2w[4 * r + 0], x0), mul_rn(c.c2w[4 * r + 1], x1));
        v[r] = add_rn(s, c.c2w[4 * r + 2]);
    }
    double n2 = add_rn(add_rn(mul_rn(v[0], v[0]), mul_rn(v[1], v[1])), mul_rn(v[2], v[2]));
    double n = __dsqrt_rn(n2);
#pragma unroll
    for (int r = 0; r < 3; r++) { d[r] = div_rn(v[r], n); o[r] = c.c2w[4 * r + 3]; }
}

// Region-boundary candidates t > t_near (faces |x_j| = 1, diagonals x_i = +-x_j), sorted
// ascending with +inf padding.  Sorting network on registers (exact min/max).
__device__ __forceinline__ void boundary_candidates(const double o[3], const double d[3],
                                                    double t_near, double cand[12]) {
    const double inf = __longlong_as_double(0x7ff0000000000000ll);
#pragma unroll
    for (int j = 0; j < 3; j++) {
        double t1 = inf, t2 = inf;
        if (d[j] != 0.0) {
            t1 = div_rn(sub_rn(1.0, o[j]), d[j]);
            t2 = div_rn(sub_rn(-1.0, o[j]), d[j]);
        }
        cand[2 * j] = t1;
        cand[2 * j + 1] = t2;
    }
    const int pi_[3] = {0, 0, 1}, pj_[3] = {1, 2, 2};
#pragma unroll
    for (int p = 0; p < 3; p++) {
        int i = pi_[p], j = pj_[p];
        double den = sub_rn(d[i], d[j]);
        double t1 = inf, t2 = inf;
        if (den != 0.0) t1 = div_rn(sub_rn(o[j], o[i]), den);
        double den2 = add_rn(d[i], d[j]);
        if (den2 != 0.0) t2 = div_rn(-add_rn(o[i], o[j]), den2);
        cand[6 + 2 * p] = t1;
        cand[7 + 2 * p] = t2;
    }
#pragma unroll
    for (int k = 0; k < 12; k++)
        if (!(cand[k] > t_near) || !isfinite(cand[k])) cand[k] = inf;
    // Batcher odd-even merge sort for 16 inputs pruned to the 12 live ones (41 exact min/max
    // compare-exchanges, fully unrolled -> registers; verified on all 2^12 0/1 inputs)
    constexpr int kNet[41][2] = {{0, 1}, {2, 3}, {0, 2}, {1, 3}, {1, 2}, {4, 5}, {6, 7}, {4, 6}, {5, 7},
                                 {5, 6}, {0, 4}, {2, 6}, {2, 4}, {1, 5}, {3, 7}, {3, 5}, {1, 2}, {3, 4},
                                 {5, 6}, {8, 9}, {10, 11}, {8, 10}, {9, 11}, {9, 10}, {0, 8}, {4, 8},
                                 {2, 10}, {6, 10}, {2, 4}, {6, 8}, {1, 9}, {5, 9}, {3, 11}, {7, 11},
                                 {3, 5}, {7, 9}, {1, 2}, {3, 4}, {5, 6}, {7, 8}, {9, 10}};
    // compare-exchange by one compare + selects: the candidates are never NaN (non-finite ones
    // were set to +inf above), so fmin/fmax's NaN handling is dead weight
#pragma unroll
    for (int c = 0; c < 41; c++) {
        const double a = cand[kNet[c][0]], b = cand[kNet[c][1]];
        const bool lt = a < b;
        cand[kNet[c][0]] = lt ? a : b;
        cand[kNet[c][1]] = lt ? b : a;
    }
}

// One contracted segment: lattice origin Qa, step U, sample count K (readings D5-D8).
struct Segment {
    int Qa[3];
    int U[3];
    int K;
    int region;
};

// Returns false if the segment has zero contracted length (dropped).
__device__ __forceinline__ bool make_segment(const DevScene& S, int g, const double o[3],
                                             const double d[3], double ta, double tb,
                                             Segment& seg) {
    double xa[3], ca[3], cb[3];
    point_at(o, d, ta, xa);
    contract_region(g, xa, ca);
    if (isinf(tb)) {
        vanishing_point(g, d, cb);
    } else {
        double xb[3];
        point_at(o, d, tb, xb);
        contract_region(g, xb, cb);
    }
    double dx[3];
#pragma unroll
    for (int q = 0; q < 3; q++) dx[q] = sub_rn(cb[q], ca[q]);
    double l2 = add_rn(add_rn(mul_rn(dx[0], dx[0]), mul_rn(dx[1], dx[1])), mul_rn(dx[2], dx[2]));
    double len = __dsqrt_rn(l2);
    if (!(len > 0.0)) return false;
#pragma unroll
    for (int q = 0; q < 3; q++) {
        double u = div_rn(dx[q], len);
        seg.Qa[q] = (int)__double2ll_rn(mul_rn(ca[q], (double)kOne));
        seg.U[q] = (int)__double2ll_rn(mul_rn(u, S.lattice_step));
    }
    seg.K = (int)ceil(mul_rn(len, S.inv_step));   // == len / Delta exactly (power of two)
    seg.region = g;
    return true;
}

// MUFU-only exp2 / reciprocal (flush-to-zero; no range fix-up instructions)
__device__ __forceinline__ float ex2_ftz(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_ftz(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// ------------------------------------------------------------------------------------
// int32 lattice helpers (F = 28: |Q| <= 2^29 + drift, so every position, cell and texel
// coordinate fits a 32-bit register)
// ------------------------------------------------------------------------------------
// Lattice positions in the kernels are BIASED by contracted 2.0: Qb = Q + 2^(F+1), so the
// contracted cube [-2, 2)^3 maps to [0, 2^(F+2)) and a cell / texel index is a plain shift.
// (The workspace segments store biased origins; merf_segment records keep the unbiased Qa.)
__device__ __forceinline__ int occ_cell(int Qb, int shift, int N) {
    int c = Qb >> shift;
    return min(max(c, 0), N - 1);
}

__device__ __forceinline__ bool occ_bit(const uint32_t* bits, int cx, int cy, int cz, int N) {
    uint32_t lin = ((uint32_t)cz * N + cy) * N + cx;
    uint32_t w = __ldg(bits + (lin >> 5));
    return (w >> (lin & 31)) & 1u;
}

constexpr float kMagicF = 12582912.f;          // 1.5 * 2^23
constexpr uint32_t kMagicBits = 0x4B400000u;   // its bit pattern (low 22 bits zero)

// First k' >= 0 with Qa + k' U outside [lo, hi) along one axis, capped at K.  Both signs
// reduce to e = ceil(num / |U|) with num = hi - Qa (U > 0) or Qa - lo + 1 (U < 0), num >= 1
// while the current sample is inside the cell; U = 0 gives +inf -> K.  The fp32 estimate is
// within one of the exact quotient (relative error ~2^-21, e <= K < 2^21), so one branch-free
// correction each way makes it exact; e |U| <= (K + 1) |U| < 2^31 (the segment's lattice
// length) cannot overflow.
__device__ __forceinline__ int exit_axis(int Qa, int U, int lo, int hi, int K) {
    const int a = abs(U);
    const int num = U > 0 ? hi - Qa : Qa - lo + 1;
    // ceil of the estimate num * rcp(a) (1 - 2^-22) in one FFMA rounding up onto the integer grid
    // of the 1.5 * 2^23 magic (exact below 2^22; positive float bit patterns are monotonic, so
    // any larger, infinite or NaN quotient (a = 0) still clamps to K): no FRND / F2I on the XU
    // pipe.  MUFU rcp is within 2^-23 of 1/a and (float)num within 2^-24 of num, so the biased
    // product is never above num / a and, for num / a < 2^21, above num / a - 1: the estimate is
    // ceil(num / a) or one less, and one upward correction makes it exact.  (Beyond 2^21 -- a
    // skip of > 2M samples, only at steps below 2^-18 -- it may land short of the exit, inside
    // the same empty cell, which the next probe skips again: never past an occupied sample.)
    const float rc = rcp_ftz((float)a) * 0.99999976158142090f;       // 1 - 2^-22
    const float t = __fmaf_ru((float)num, rc, kMagicF);
    int e = min((int)(__float_as_uint(t) - kMagicBits), K);
    e += (e * a < num) ? 1 : 0;
    return min(e, K);
}

// texel coordinate on a grid of resolution M = 2^m (s = F + 2 - m): lower index, fraction
// (cell-centred texels, clamp to edge; reading D9).  The position is clamped at texel 0 only:
// past the centre of texel M-1 (the last half texel of the contracted cube, and lattice drift)
// i0 = M-1 with 0 < f <= 1/2 + drift, and corner i0 + 1 = M is stored as a copy of texel M-1
// in every layout (the planes' extra row per plane and pair entry (M-1, M-1), the atlas apron
// of edge blocks, made to replicate the edge at upload).  The integer weights of the two
// corners sum to their parent exactly, so this is bit-identical to clamping the position to
// texel M-1 (f = 0), without the min on every axis of every sample.
__device__ __forceinline__ void texel(int Qb, int s, int M, int& i0, float& f) {
    (void)M;
    const int P = max(Qb - (1 << (s - 1)), 0);
    i0 = P >> s;
    f = (float)(P & ((1 << s) - 1)) * __int_as_float((127 - s) << 23);
}

// The same texel coordinate with the fraction delivered as g = 2^23 + f 2^s, an exact float
// built by one LOP3 (needs s <= 23; the compile-time paper geometry has s = 21, 19): no I2F and
// no scaling multiply.  g_frac recovers f exactly (power-of-two scaling, one FFMA).
// MERF_BOUNDS_CHECK builds (tests / stress only): every gathered index is checked against its
// buffer and a violation traps (compute-sanitizer is unavailable on the GPU pool)
#ifdef MERF_BOUNDS_CHECK
#define MERF_CHECK(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define MERF_CHECK(cond) do { } while (0)
#endif

__device__ __forceinline__ float exp2i(int n) { return __int_as_float((127 + n) << 23); }
__device__ __forceinline__ void texel_g(int Qb, int s, int M, int& i0, float& g) {
    (void)M;
    const int P = max(Qb - (1 << (s - 1)), 0);        // upper edge: see texel()
    i0 = P >> s;
    unsigned b;                        // (P & mask) | 0x4B000000 in one LOP3
    asm("lop3.b32 %0, %1, %2, %3, 0xea;" : "=r"(b) : "r"(P), "r"((1 << s) - 1), "r"(0x4B000000));
    g = __uint_as_float(b);
}
__device__ __forceinline__ float g_frac(float g, int s) { return fmaf(g, exp2i(-s), -exp2i(23 - s)); }

// 16-bit fixed-point interpolation weights that partition 65535 EXACTLY (so a constant
// field interpolates exactly): split an integer weight W along one axis with fraction f
// into (W - round(f W), round(f W)).  The rounding is one FFMA against the 1.5 * 2^23 magic
// (t = f W + M leaves round(f W) in the low mantissa bits: no F2I), and every weight is
// carried both as an int and as an exact float so the next split needs no conversion.
//
// Integer weights that feed a LEAF split are carried BIASED, Wb = W - 65535 M (mod 2^32), so the
// leaf packs its dp2a operand with one IMAD: with t = M + w1 (bits of the leaf's FFMA),
// 65535 t + Wb = W + 65535 w1 = (W - w1) + (w1 << 16) -- lo16 = W - w1, hi16 = w1 (both in
// [0, 65535], no carry).  B selects the biased form of a split's two children.
constexpr uint32_t kLeafBias = 65535u * kMagicBits;   // mod 2^32
template <bool B = false>
__device__ __forceinline__ void wsplit(uint32_t Wi, float Wf, float f, uint32_t& w0i, float& w0f, uint32_t& w1i,
                                       float& w1f) {
    const float t = fmaf(f, Wf, kMagicF);
    const uint32_t tb = __float_as_uint(t);
    w1i = tb - (kMagicBits + (B ? kLeafBias : 0u));
    w0i = Wi - tb + (kMagicBits - (B ? kLeafBias : 0u));
    w1f = t - kMagicF;
    w0f = Wf - w1f;
}
// the first split of the full weight 65535 straight from g: f 65535 + M = g (65535 2^-s) +
// (M - 65535 2^(23-s)), both constants exact, so t is bit-identical to wsplit's
template <bool B = false>
__device__ __forceinline__ void wsplit_full_g(float g, int s, uint32_t& w0i, float& w0f, uint32_t& w1i, float& w1f) {
    const float t = fmaf(g, 65535.f * exp2i(-s), kMagicF - 65535.f * exp2i(23 - s));
    const uint32_t tb = __float_as_uint(t);
    w1i = tb - (kMagicBits + (B ? kLeafBias : 0u));
    w0i = (65535u + kMagicBits - (B ? kLeafBias : 0u)) - tb;
    w1f = t - kMagicF;
    w0f = 65535.f - w1f;
}
// the last split of a BIASED weight Wb, packed as the (lo16, hi16) = (W - w1, w1) operand of
// dp2a: FFMA + IMAD (the multiply-add runs on the FMA pipe; the ALU pipe is the march's
// busiest)
__device__ __forceinline__ uint32_t wleaf(uint32_t Wb, float Wf, float f) {
    const uint32_t t = __float_as_uint(fmaf(f, Wf, kMagicF));   // kMagicBits + w1
    return t * 65535u + Wb;
}

}  // namespace merf
