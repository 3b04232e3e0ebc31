/*
 * merf_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, fp64 CPU renderer of a baked MERF scene, written directly from the
 * paper (arXiv 2302.12249, /root/reference/PAPER.md, cited as P:<line>).  It is the
 * parity oracle for the CUDA path and the `cpu_baseline` of bench.py.  Only tests/,
 * __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may load it.
 * It shares no code, header, table or constant generator with
 * paper_2302_12249_b200/ and never calls it.
 *
 * Every function cites the passage it follows.  Where the paper is silent the reading
 * from DESIGN.md section "Readings" (D1..D22) is named.  Arithmetic is IEEE binary64,
 * compiled with -O2 -ffp-contract=off (no FMA contraction, no fast-math), evaluated in
 * the canonical operation order written out in DESIGN.md "Canonical fp64 setup" (D8).
 *
 * Parity pins: see tests/test_oracle_*.py.  Functions whose numerical convention is a
 * reading rather than a paper fact (direction-encoding order D17, texel placement D9,
 * delta convention D4) are "parity unpinned vs the paper" and say so below.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_F 28                          /* fixed-point fraction bits of the lattice (D8) */
#define ORC_ONE ((int64_t)1 << ORC_F)     /* contracted 1.0 in lattice units              */
#define ORC_TWO ((int64_t)1 << (ORC_F + 1)) /* contracted 2.0                              */
#define ORC_MAXSEG 16

/* ---------------------------------------------------------------------------------- */
/* Scene as seen by the oracle (host arrays owned by the caller).                      */
/* ---------------------------------------------------------------------------------- */
typedef struct {
    int32_t L;              /* 3D grid resolution, 0 = no grid */
    int32_t R;              /* plane resolution, 0 = no planes */
    int32_t C;              /* channels = 8 */
    int32_t n_levels;       /* occupancy levels, coarse -> fine */
    int32_t level_res[4];
    double m_density;       /* 14 */
    double m_appearance;    /* 7 */
    double step;            /* uniform contracted step Delta (D5) */
    double t_min;           /* termination transmittance 2e-4 */
    double alpha_skip;      /* appearance read iff alpha > alpha_skip (D14) */
    uint32_t source_mask;   /* bit0 V, bit1 P_x, bit2 P_y, bit3 P_z                       */
    const uint8_t *planes;  /* [3][R][R][C]: P_x[z][y], P_y[z][x], P_z[y][x]             */
    const int32_t *block_index; /* [(L/8)^3] raster (z,y,x), -1 = not stored */
    const uint8_t *atlas;   /* [n_blocks][9][9][9][C] (z,y,x), 1-voxel apron on + side   */
    int64_t n_blocks;
    const uint32_t *occ[4]; /* occupancy bits per level, x fastest, LSB first */
    const double *mlp;      /* 883: W0[16][34] b0[16] W1[16][16] b1[16] W2[3][16] b2[3]  */
} orc_scene;

typedef struct {
    int32_t region;         /* 0 core, 1+2j+(s<0) for outer region (j,s)                 */
    int32_t ordinal;        /* index among kept segments                                 */
    double t_a, t_b;        /* world ray parameter interval (t_b may be +inf)            */
    double c_a[3], c_b[3];  /* contracted endpoints                                      */
    double len;             /* contracted length l                                       */
    double u[3];            /* contracted unit direction                                 */
    int64_t Qa[3];          /* lattice origin llrint(c_a * 2^F)                          */
    int64_t U[3];           /* lattice step llrint(u * Delta * 2^F)                      */
    int64_t K;              /* number of samples ceil(l / Delta)                         */
} orc_segment;

/* ---------------------------------------------------------------------------------- */
/* Contraction (Sec. 4.2).                                                  */
/* ---------------------------------------------------------------------------------- */

/* region_of: CORE iff ||x||_inf <= 1 (read as <= 1, D2); otherwise the coordinate
 * j maximising |x_j| (first such index on ties, D1) and its sign. */
int orc_region_of(const double x[3])
{
    double ax = fabs(x[0]), ay = fabs(x[1]), az = fabs(x[2]);
    double m = ax;
    if (ay > m) m = ay;
    if (az > m) m = az;
    if (m <= 1.0) return 0;
    int j = (ax == m) ? 0 : ((ay == m) ? 1 : 2);
    return 1 + 2 * j + (x[j] < 0.0 ? 1 : 0);
}

/* contract_pi evaluated with region g's formula:
 *   core: identity; (j,s): c_j = s (2 - 1/|x_j|), c_k = x_k / |x_j|. */
void orc_contract_region(int g, const double x[3], double c[3])
{
    if (g == 0) { c[0] = x[0]; c[1] = x[1]; c[2] = x[2]; return; }
    int j = (g - 1) / 2;
    int neg = (g - 1) % 2;
    double a = fabs(x[j]);
    for (int k = 0; k < 3; k++) {
        if (k == j) {
            double r = 1.0 / a;
            double v = 2.0 - r;
            c[k] = neg ? -v : v;
        } else {
            c[k] = x[k] / a;
        }
    }
}

/* contract_pi(x) for arrays: y[i] = contract_pi(x[i]), region[i] = region_of(x[i]). */
void orc_contract(const double *x, int64_t n, double *y, int32_t *region)
{
    for (int64_t i = 0; i < n; i++) {
        int g = orc_region_of(x + 3 * i);
        if (region) region[i] = g;
        orc_contract_region(g, x + 3 * i, y + 3 * i);
    }
}

/* Limit of contract_g(o + t d) as t -> inf in outer region g=(j,s): c_j = 2s, c_k = d_k/|d_j|. */
static void orc_vanishing_point(int g, const double d[3], double c[3])
{
    int j = (g - 1) / 2;
    int neg = (g - 1) % 2;
    double a = fabs(d[j]);
    for (int k = 0; k < 3; k++) {
        if (k == j) c[k] = neg ? -2.0 : 2.0;
        else c[k] = d[k] / a;
    }
}

/* ---------------------------------------------------------------------------------- */
/* Camera rays (P:140 x = o + t d; pinhole model reading D18).                         */
/* cam = [c2w row-major 3x4 (12), fx, fy, cx, cy, t_near].                              */
/* ---------------------------------------------------------------------------------- */
void orc_raygen(const double *cam, int32_t i, int32_t j, double o[3], double d[3])
{
    double a0 = (double)i + 0.5;
    double a1 = (double)j + 0.5;
    double x0 = (a0 - cam[14]) / cam[12];
    double x1 = (a1 - cam[15]) / cam[13];
    double v[3];
    for (int r = 0; r < 3; r++) {
        double p = cam[4 * r + 0] * x0;
        double q = cam[4 * r + 1] * x1;
        double s = p + q;
        v[r] = s + cam[4 * r + 2];
    }
    double n2 = v[0] * v[0] + v[1] * v[1];
    n2 = n2 + v[2] * v[2];
    double n = sqrt(n2);
    for (int r = 0; r < 3; r++) { d[r] = v[r] / n; o[r] = cam[4 * r + 3]; }
}

/* ---------------------------------------------------------------------------------- */
/* Ray segmentation into regions ("The origin and direction of a ray can        */
/* therefore be computed in contracted space"; readings D3, D6, D8).                   */
/* ---------------------------------------------------------------------------------- */
static int cmp_double(const void *a, const void *b)
{
    double x = *(const double *)a, y = *(const double *)b;
    return (x < y) ? -1 : ((x > y) ? 1 : 0);
}

static void point_at(const double o[3], const double d[3], double t, double x[3])
{
    for (int k = 0; k < 3; k++) { double p = t * d[k]; x[k] = o[k] + p; }
}

/* Returns the number of kept segments written to seg (<= ORC_MAXSEG). */
int orc_segment_ray(const double o[3], const double d[3], double t_near, double step,
                    orc_segment *seg)
{
    /* candidate boundaries: faces |x_j| = 1 and diagonals x_i = +-x_j */
    double cand[12];
    int nc = 0;
    for (int j = 0; j < 3; j++) {
        if (d[j] != 0.0) {
            double t1 = (1.0 - o[j]) / d[j];
            double t2 = (-1.0 - o[j]) / d[j];
            cand[nc++] = t1;
            cand[nc++] = t2;
        }
    }
    static const int pi_[3] = {0, 0, 1}, pj_[3] = {1, 2, 2};
    for (int p = 0; p < 3; p++) {
        int i = pi_[p], j = pj_[p];
        double den = d[i] - d[j];
        if (den != 0.0) cand[nc++] = (o[j] - o[i]) / den;
        double den2 = d[i] + d[j];
        if (den2 != 0.0) { double s = o[i] + o[j]; cand[nc++] = (-s) / den2; }
    }
    /* keep t > t_near, finite; sort ascending; unique */
    double b[14];
    int nb = 0;
    b[nb++] = t_near;
    qsort(cand, nc, sizeof(double), cmp_double);
    for (int k = 0; k < nc; k++) {
        double t = cand[k];
        if (!(t > t_near) || !isfinite(t)) continue;
        if (t == b[nb - 1]) continue;
        b[nb++] = t;
    }
    /* region of every interval [b_i, b_{i+1}] (last interval unbounded) */
    int reg[14];
    for (int k = 0; k < nb; k++) {
        double p;
        if (k + 1 < nb) { double s = b[k] + b[k + 1]; p = s * 0.5; }
        else { double s = b[k] * 2.0; p = s + 1.0; }
        double x[3];
        point_at(o, d, p, x);
        reg[k] = orc_region_of(x);
    }
    /* merge equal neighbours, contract endpoints, lattice setup */
    int ns = 0;
    int k = 0;
    while (k < nb) {
        int g = reg[k];
        int e = k;
        while (e + 1 < nb && reg[e + 1] == g) e++;
        double ta = b[k];
        double tb = (e + 1 < nb) ? b[e + 1] : INFINITY;
        orc_segment S;
        memset(&S, 0, sizeof(S));
        S.region = g;
        S.t_a = ta;
        S.t_b = tb;
        double xa[3];
        point_at(o, d, ta, xa);
        orc_contract_region(g, xa, S.c_a);
        if (isinf(tb)) {
            orc_vanishing_point(g, d, S.c_b);
        } else {
            double xb[3];
            point_at(o, d, tb, xb);
            orc_contract_region(g, xb, S.c_b);
        }
        double dx[3];
        for (int q = 0; q < 3; q++) dx[q] = S.c_b[q] - S.c_a[q];
        double l2 = dx[0] * dx[0] + dx[1] * dx[1];
        l2 = l2 + dx[2] * dx[2];
        double len = sqrt(l2);
        k = e + 1;
        if (!(len > 0.0)) continue; /* zero-length segment dropped */
        S.len = len;
        double scale = step * (double)ORC_ONE; /* Delta * 2^F, exact (Delta power of two) */
        for (int q = 0; q < 3; q++) {
            S.u[q] = dx[q] / len;
            S.Qa[q] = llrint(S.c_a[q] * (double)ORC_ONE);
            S.U[q] = llrint(S.u[q] * scale);
        }
        S.K = (int64_t)ceil(len / step);
        S.ordinal = ns;
        if (ns < ORC_MAXSEG) seg[ns++] = S;
    }
    return ns;
}

/* ---------------------------------------------------------------------------------- */
/* Occupancy pyramid: max-pooling of the finest binary grid.           */
/* ---------------------------------------------------------------------------------- */
static int get_bit(const uint32_t *bits, int64_t lin)
{
    return (int)((bits[lin >> 5] >> (lin & 31)) & 1u);
}

/* coarse[N^3 bits] = max over each (f/N)^3 block of fine[f^3 bits]; literal loops. */
void orc_maxpool_bits(const uint32_t *fine, int32_t f, uint32_t *coarse, int32_t N)
{
    int64_t words = ((int64_t)N * N * N + 31) / 32;
    memset(coarse, 0, (size_t)words * 4);
    int r = f / N;
    for (int z = 0; z < N; z++)
        for (int y = 0; y < N; y++)
            for (int x = 0; x < N; x++) {
                int any = 0;
                for (int dz = 0; dz < r && !any; dz++)
                    for (int dy = 0; dy < r && !any; dy++)
                        for (int dx = 0; dx < r && !any; dx++) {
                            int64_t lin = ((int64_t)(z * r + dz) * f + (y * r + dy)) * f + (x * r + dx);
                            if (get_bit(fine, lin)) any = 1;
                        }
                if (any) {
                    int64_t lin = ((int64_t)z * N + y) * N + x;
                    coarse[lin >> 5] |= 1u << (lin & 31);
                }
            }
}

/* ---------------------------------------------------------------------------------- */
/* Lattice -> grid coordinates.  Cell-centred texels, spacing 4/M, clamp to edge (D9). */
/* ---------------------------------------------------------------------------------- */
static int ilog2i(int64_t v) { int n = 0; while (((int64_t)1 << n) < v) n++; return n; }

/* occupancy cell index at resolution N for lattice coordinate Q (D10): the cell of
 * [-2, 2) split into N equal half-open cells that contains Q 2^-F, clamped to [0, N-1]
 * (pinned against real arithmetic in tests/test_oracle_lattice.py) */
static int64_t occ_cell(int64_t Q, int32_t N)
{
    int s = ORC_F + 2 - ilog2i(N);
    int64_t c = (Q + ORC_TWO) >> s;
    if (c < 0) c = 0;
    if (c > N - 1) c = N - 1;
    return c;
}

/* exported for the pins only */
int64_t orc_occ_cell(int64_t Q, int32_t N) { return occ_cell(Q, N); }

/* lower texel index i0 and fraction f of coordinate Q on a grid of resolution M */
static void texel_coord(int64_t Q, int32_t M, int64_t *i0, double *f)
{
    int m = ilog2i(M);
    int s = ORC_F + 2 - m;
    int64_t half = (int64_t)1 << (s - 1);
    int64_t P = Q + ORC_TWO - half;
    int64_t i = P >> s;
    int64_t rem = P - (i << s);
    double fr = (double)rem / (double)((int64_t)1 << s);
    if (i < 0) { i = 0; fr = 0.0; }
    if (i > M - 2) { i = M - 2; fr = 1.0; }
    *i0 = i;
    *f = fr;
}

/* ---------------------------------------------------------------------------------- */
/* Canonical block allocation ("only store data blocks that contain occupied    */
/* voxels"; reading D11): block b is needed iff some occupied cell of the finest level */
/* can produce a sample whose trilinear base voxel i0 lies in b.  Raster numbering.    */
/* ---------------------------------------------------------------------------------- */
int64_t orc_canonical_block_index(const uint32_t *finest, int32_t N, int32_t L, int32_t *index_out)
{
    int nb = L / 8;
    int64_t slots = (int64_t)nb * nb * nb;
    uint8_t *need = (uint8_t *)calloc((size_t)slots, 1);
    int s = ORC_F + 2 - ilog2i(N);
    for (int z = 0; z < N; z++)
        for (int y = 0; y < N; y++)
            for (int x = 0; x < N; x++) {
                int64_t lin = ((int64_t)z * N + y) * N + x;
                if (!get_bit(finest, lin)) continue;
                int cc[3] = {x, y, z};
                int64_t blo[3], bhi[3];
                for (int a = 0; a < 3; a++) {
                    /* i0 is monotone in Q; edge cells also cover the clamped outside */
                    int64_t lo_i, hi_i;
                    double fdum;
                    if (cc[a] == 0) lo_i = 0;
                    else texel_coord(((int64_t)cc[a] << s) - ORC_TWO, L, &lo_i, &fdum);
                    if (cc[a] == N - 1) hi_i = L - 2;
                    else texel_coord((((int64_t)cc[a] + 1) << s) - ORC_TWO - 1, L, &hi_i, &fdum);
                    blo[a] = lo_i >> 3;
                    bhi[a] = hi_i >> 3;
                }
                for (int64_t bz = blo[2]; bz <= bhi[2]; bz++)
                    for (int64_t by = blo[1]; by <= bhi[1]; by++)
                        for (int64_t bx = blo[0]; bx <= bhi[0]; bx++)
                            need[(bz * nb + by) * nb + bx] = 1;
            }
    int64_t n = 0;
    for (int64_t i = 0; i < slots; i++) index_out[i] = need[i] ? (int32_t)(n++) : -1;
    free(need);
    return n;
}

/* ---------------------------------------------------------------------------------- */
/* Field query (Eq. 5, Fig. 2; dequantisation Eq. 7, D13).      */
/* Each stored byte is decoded to 2m*b/255 - m, then interpolated, then the four      */
/* sources are summed.  Returns the number of missing V blocks hit (0 for sound).     */
/* ---------------------------------------------------------------------------------- */
static double dequant(uint8_t b, double m)
{
    double v = 2.0 * m * (double)b;
    return v / 255.0 - m;
}

int orc_query_field(const orc_scene *S, const int64_t Q[3], double t[8])
{
    int C = S->C;
    int missing = 0;
    for (int c = 0; c < C; c++) t[c] = 0.0;
    double mch[8];
    for (int c = 0; c < C; c++) mch[c] = (c == 0) ? S->m_density : S->m_appearance;

    double v[8] = {0};
    if ((S->source_mask & 1u) && S->L > 0) {
        int64_t i0[3];
        double f[3];
        for (int a = 0; a < 3; a++) texel_coord(Q[a], S->L, &i0[a], &f[a]);
        int nb = S->L / 8;
        int64_t slot = ((i0[2] >> 3) * nb + (i0[1] >> 3)) * nb + (i0[0] >> 3);
        int32_t blk = S->block_index[slot];
        if (blk < 0 || blk >= S->n_blocks) {
            missing = 1; /* contributes nothing (soundness violation, counted) */
        } else {
            const uint8_t *base = S->atlas + (size_t)blk * 729 * C;
            for (int dz = 0; dz < 2; dz++)
                for (int dy = 0; dy < 2; dy++)
                    for (int dx = 0; dx < 2; dx++) {
                        double w = (dx ? f[0] : 1.0 - f[0]) * (dy ? f[1] : 1.0 - f[1]);
                        w = w * (dz ? f[2] : 1.0 - f[2]);
                        int lx = (int)(i0[0] & 7) + dx, ly = (int)(i0[1] & 7) + dy, lz = (int)(i0[2] & 7) + dz;
                        const uint8_t *texel = base + ((size_t)(lz * 9 + ly) * 9 + lx) * C;
                        for (int c = 0; c < C; c++) v[c] += w * dequant(texel[c], mch[c]);
                    }
        }
    }
    double p[3][8] = {{0}};
    if (S->R > 0) {
        /* plane a is perpendicular to axis a: P_x(y,z), P_y(x,z), P_z(x,y) */
        static const int ua[3] = {1, 0, 0}, va[3] = {2, 2, 1};
        for (int a = 0; a < 3; a++) {
            if (!(S->source_mask & (2u << a))) continue;
            int64_t iu, iv;
            double fu, fv;
            texel_coord(Q[ua[a]], S->R, &iu, &fu);
            texel_coord(Q[va[a]], S->R, &iv, &fv);
            const uint8_t *pl = S->planes + (size_t)a * S->R * S->R * C;
            for (int dv = 0; dv < 2; dv++)
                for (int du = 0; du < 2; du++) {
                    double w = (du ? fu : 1.0 - fu) * (dv ? fv : 1.0 - fv);
                    const uint8_t *texel = pl + ((size_t)(iv + dv) * S->R + (size_t)(iu + du)) * C;
                    for (int c = 0; c < C; c++) p[a][c] += w * dequant(texel[c], mch[c]);
                }
        }
    }
    for (int c = 0; c < C; c++) {
        double s = v[c] + p[0][c];
        s = s + p[1][c];
        t[c] = s + p[2][c];
    }
    return missing;
}

/* ---------------------------------------------------------------------------------- */
/* Deferred MLP h (Eq. 3; 3 layers, 16 hidden, 4 frequencies P:580;        */
/* ReLU/ReLU/sigmoid and encoding order are readings D16-D17: parity unpinned vs paper)*/
/* ---------------------------------------------------------------------------------- */
static double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }

void orc_encode_dir(const double d[3], double enc[27])
{
    enc[0] = d[0]; enc[1] = d[1]; enc[2] = d[2];
    int n = 3;
    for (int j = 0; j < 3; j++)
        for (int k = 0; k < 4; k++) {
            double a = ldexp(d[j], k);
            enc[n++] = sin(a);
            enc[n++] = cos(a);
        }
}

void orc_mlp(const double *w, const double cd[3], const double F[4], const double d[3], double h[3])
{
    double x[34];
    x[0] = cd[0]; x[1] = cd[1]; x[2] = cd[2];
    x[3] = F[0]; x[4] = F[1]; x[5] = F[2]; x[6] = F[3];
    orc_encode_dir(d, x + 7);
    const double *W0 = w, *b0 = w + 544, *W1 = w + 560, *b1 = w + 816, *W2 = w + 832, *b2 = w + 880;
    double h0[16], h1[16];
    for (int o = 0; o < 16; o++) {
        double s = b0[o];
        for (int i = 0; i < 34; i++) s += W0[o * 34 + i] * x[i];
        h0[o] = s > 0.0 ? s : 0.0;
    }
    for (int o = 0; o < 16; o++) {
        double s = b1[o];
        for (int i = 0; i < 16; i++) s += W1[o * 16 + i] * h0[i];
        h1[o] = s > 0.0 ? s : 0.0;
    }
    for (int o = 0; o < 3; o++) {
        double s = b2[o];
        for (int i = 0; i < 16; i++) s += W2[o * 16 + i] * h1[i];
        h[o] = sigmoid(s);
    }
}

/* ---------------------------------------------------------------------------------- */
/* Ray march (Eq. 1-3; occupancy traversal P:307-309; texture split P:311). */
/* mode 0: hierarchical coarse-to-fine skipping with lattice-snapped AABB exits (D7). */
/* mode 1: dense stepping, every lattice sample gated by the finest level only.       */
/* ---------------------------------------------------------------------------------- */
#define ORC_NO_EARLY_TERM 1u

typedef struct {
    double rgb[3];
    double cd[3], F[4], T;
    int64_t n_eval, n_density_only, n_skip, n_missing;
    int32_t n_seg;
    int32_t region_mask;
} orc_ray_result;

static int64_t floor_div(int64_t a, int64_t b) /* b > 0 */
{
    int64_t q = a / b;
    if ((a % b != 0) && (a < 0)) q -= 1;
    return q;
}
static int64_t ceil_div(int64_t a, int64_t b) /* b > 0 */
{
    return -floor_div(-a, b);
}

/* first k' at which sample Qa + k' U leaves cell `cell` (res N) along any axis */
static int64_t exit_index(const int64_t Qa[3], const int64_t U[3], const int64_t cell[3], int32_t N)
{
    int s = ORC_F + 2 - ilog2i(N);
    int64_t best = INT64_MAX;
    for (int a = 0; a < 3; a++) {
        int64_t face_lo = (cell[a] << s) - ORC_TWO;
        int64_t face_hi = ((cell[a] + 1) << s) - ORC_TWO;
        int64_t e;
        if (U[a] > 0) e = ceil_div(face_hi - Qa[a], U[a]);
        else if (U[a] < 0) e = floor_div(Qa[a] - face_lo, -U[a]) + 1;
        else continue;
        if (e < best) best = e;
    }
    return best;
}

void orc_march(const orc_scene *S, const double o[3], const double d[3], double t_near, int mode,
               uint32_t flags, orc_ray_result *res, int32_t max_trace, uint64_t *trace_cells,
               double *trace_T, int32_t *trace_count)
{
    orc_segment seg[ORC_MAXSEG];
    int ns = orc_segment_ray(o, d, t_near, S->step, seg);
    double T = 1.0, cd[3] = {0, 0, 0}, F[4] = {0, 0, 0, 0};
    int64_t n_eval = 0, n_donly = 0, n_skip = 0, n_missing = 0;
    int32_t ntr = 0;
    int done = 0;
    int32_t rmask = 0;
    int nl = S->n_levels;
    int32_t Nf = S->level_res[nl - 1];
    for (int si = 0; si < ns; si++) rmask |= 1 << seg[si].region;
    for (int si = 0; si < ns && !done; si++) {
        const orc_segment *g = &seg[si];
        int64_t k = 0;
        while (k < g->K && !done) {
            int64_t Q[3];
            for (int a = 0; a < 3; a++) Q[a] = g->Qa[a] + k * g->U[a];
            int occupied = 1;
            if (mode == 1) {
                int64_t c[3];
                for (int a = 0; a < 3; a++) c[a] = occ_cell(Q[a], Nf);
                occupied = get_bit(S->occ[nl - 1], (c[2] * Nf + c[1]) * Nf + c[0]);
                if (!occupied) { k++; continue; }
            } else {
                for (int lev = 0; lev < nl; lev++) {
                    int32_t N = S->level_res[lev];
                    int64_t c[3];
                    for (int a = 0; a < 3; a++) c[a] = occ_cell(Q[a], N);
                    if (!get_bit(S->occ[lev], (c[2] * N + c[1]) * N + c[0])) {
                        int64_t e = exit_index(g->Qa, g->U, c, N);
                        int64_t kn = k + 1;
                        if (e > kn) kn = e;
                        if (kn > g->K) kn = g->K;
                        k = kn;
                        n_skip++;
                        occupied = 0;
                        break;
                    }
                }
                if (!occupied) continue;
            }
            /* evaluate sample k (Eq. 5-6, Eq. 1-2) */
            double t[8];
            n_missing += orc_query_field(S, Q, t);
            double tau = exp(t[0]);
            double alpha = 1.0 - exp(-(tau * S->step));
            n_eval++;
            if (alpha > S->alpha_skip) {
                double w = alpha * T;
                for (int c = 0; c < 3; c++) cd[c] += w * sigmoid(t[1 + c]);
                for (int c = 0; c < 4; c++) F[c] += w * sigmoid(t[4 + c]);
            } else {
                n_donly++;
            }
            T = T * (1.0 - alpha);
            if (trace_cells && ntr < max_trace) {
                int64_t c[3];
                for (int a = 0; a < 3; a++) c[a] = occ_cell(Q[a], Nf);
                uint64_t cell = (uint64_t)((c[2] * Nf + c[1]) * Nf + c[0]);
                trace_cells[ntr] = ((uint64_t)g->ordinal << 61) | ((uint64_t)k << 40) | cell;
                trace_T[ntr] = T;
            }
            ntr++;
            if (!(flags & ORC_NO_EARLY_TERM) && T < S->t_min) done = 1;
            k++;
        }
    }
    double h[3];
    orc_mlp(S->mlp, cd, F, d, h);
    for (int c = 0; c < 3; c++) {
        double v = cd[c] + h[c];
        res->rgb[c] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
        res->cd[c] = cd[c];
    }
    for (int c = 0; c < 4; c++) res->F[c] = F[c];
    res->T = T;
    res->n_eval = n_eval;
    res->n_density_only = n_donly;
    res->n_skip = n_skip;
    res->n_missing = n_missing;
    res->n_seg = ns;
    res->region_mask = rmask;
    if (trace_count) *trace_count = ntr;
}

void orc_march_sph(const orc_scene *S, const double o[3], const double d[3], double t_near,
                   uint32_t flags, orc_ray_result *res, int32_t max_trace, uint64_t *trace_cells,
                   double *trace_T, int32_t *trace_count);

static void orc_march_any(const orc_scene *S, const double o[3], const double d[3], double t_near, int mode,
                          uint32_t flags, orc_ray_result *res, int32_t max_trace, uint64_t *trace_cells,
                          double *trace_T, int32_t *trace_count)
{
    if (mode == 2) orc_march_sph(S, o, d, t_near, flags, res, max_trace, trace_cells, trace_T, trace_count);
    else orc_march(S, o, d, t_near, mode, flags, res, max_trace, trace_cells, trace_T, trace_count);
}

/* ---------------------------------------------------------------------------------- */
/* Image / pixel-list renderers (mode 0 hierarchical, 1 dense, 2 spherical NEXT-2).  stats (optional, int64[6]): rays, segments, evals,  */
/* density-only, skips, missing.                                                       */
/* ---------------------------------------------------------------------------------- */
void orc_render_pixels(const orc_scene *S, const double *cam, int32_t W, const int64_t *pixel_ids,
                       int64_t n, int mode, uint32_t flags, double *rgb, double *aux /* [n][8] cd,F,T or NULL */,
                       int32_t max_trace, uint64_t *trace_cells, double *trace_T, int32_t *trace_count,
                       int64_t *stats, int32_t *region_masks, int32_t n_threads)
{
    int64_t st[6] = {0, 0, 0, 0, 0, 0};
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#endif
#pragma omp parallel
    {
        int64_t lst[6] = {0, 0, 0, 0, 0, 0};
#pragma omp for schedule(dynamic, 64)
        for (int64_t r = 0; r < n; r++) {
            int32_t i = (int32_t)(pixel_ids[r] % W), j = (int32_t)(pixel_ids[r] / W);
            double o[3], d[3];
            orc_raygen(cam, i, j, o, d);
            orc_ray_result res;
            orc_march_any(S, o, d, cam[16], mode, flags, &res, max_trace,
                      trace_cells ? trace_cells + r * max_trace : NULL,
                      trace_T ? trace_T + r * max_trace : NULL,
                      trace_count ? trace_count + r : NULL);
            for (int c = 0; c < 3; c++) rgb[3 * r + c] = res.rgb[c];
            if (aux) {
                for (int c = 0; c < 3; c++) aux[8 * r + c] = res.cd[c];
                for (int c = 0; c < 4; c++) aux[8 * r + 3 + c] = res.F[c];
                aux[8 * r + 7] = res.T;
            }
            if (region_masks) region_masks[r] = res.region_mask;
            lst[0] += 1; lst[1] += res.n_seg; lst[2] += res.n_eval;
            lst[3] += res.n_density_only; lst[4] += res.n_skip; lst[5] += res.n_missing;
        }
#pragma omp critical
        for (int q = 0; q < 6; q++) st[q] += lst[q];
    }
    if (stats) for (int q = 0; q < 6; q++) stats[q] = st[q];
}

/* rays given explicitly (o, d: [n][3]) -- used for special-case pins */
void orc_render_rays(const orc_scene *S, const double *o, const double *d, const double *t_near,
                     int64_t n, int mode, uint32_t flags, double *rgb, double *aux,
                     int32_t max_trace, uint64_t *trace_cells, double *trace_T, int32_t *trace_count,
                     int64_t *stats)
{
    int64_t st[6] = {0, 0, 0, 0, 0, 0};
    for (int64_t r = 0; r < n; r++) {
        orc_ray_result res;
        orc_march_any(S, o + 3 * r, d + 3 * r, t_near ? t_near[r] : 0.0, mode, flags, &res, max_trace,
                  trace_cells ? trace_cells + r * max_trace : NULL,
                  trace_T ? trace_T + r * max_trace : NULL,
                  trace_count ? trace_count + r : NULL);
        for (int c = 0; c < 3; c++) rgb[3 * r + c] = res.rgb[c];
        if (aux) {
            for (int c = 0; c < 3; c++) aux[8 * r + c] = res.cd[c];
            for (int c = 0; c < 4; c++) aux[8 * r + 3 + c] = res.F[c];
            aux[8 * r + 7] = res.T;
        }
        st[0] += 1; st[1] += res.n_seg; st[2] += res.n_eval;
        st[3] += res.n_density_only; st[4] += res.n_skip; st[5] += res.n_missing;
    }
    if (stats) for (int q = 0; q < 6; q++) stats[q] = st[q];
}

int32_t orc_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---------------------------------------------------------------------------------- */
/* Baking (NEXT-1).                                                          */
/* "We mark the eight voxels surrounding a given point x_i as occupied if both the     */
/* volume rendering weight w_i and the opacity alpha_i exceed a threshold set to 0.005"*/
/* (P:270), alpha_i = 1 - exp(-tau_i delta) with the renderer's step.       */
/* The comparison alpha > 0.005 is taken as tau > tau_thr, tau_thr = -ln(1-0.005)/delta */
/* (monotone; the caller passes tau_thr so both implementations compare the same fp64   */
/* constant).  Points are world positions, contracted with contract_pi,     */
/* put on the 2^-F lattice and mapped to the cell-centred grid of resolution N (D9):    */
/* the eight voxels are the trilinear corners i0, i0 + 1 per axis, clamped to the grid. */
/* ---------------------------------------------------------------------------------- */
void orc_bake_occupancy(const double *x, const double *tau, const double *w, int64_t n,
                        double tau_thr, double w_thr, int32_t N, uint32_t *bits)
{
    int64_t words = ((int64_t)N * N * N + 31) / 32;
    memset(bits, 0, (size_t)words * 4);
    for (int64_t i = 0; i < n; i++) {
        if (!(w[i] > w_thr) || !(tau[i] > tau_thr)) continue;
        double c[3];
        int g = orc_region_of(x + 3 * i);
        orc_contract_region(g, x + 3 * i, c);
        int64_t lo[3], hi[3];
        for (int a = 0; a < 3; a++) {
            int64_t Q = llrint(c[a] * (double)ORC_ONE);
            int64_t i0;
            double f;
            texel_coord(Q, N, &i0, &f);
            lo[a] = i0;
            hi[a] = i0 + 1;
        }
        for (int64_t z = lo[2]; z <= hi[2]; z++)
            for (int64_t y = lo[1]; y <= hi[1]; y++)
                for (int64_t xx = lo[0]; xx <= hi[0]; xx++) {
                    int64_t lin = (z * N + y) * N + xx;
                    bits[lin >> 5] |= 1u << (lin & 31);
                }
    }
}

/* Block-sparse storage of V (reading D11): block b of the canonical/any index gets
 * the dense grid's voxels 8b .. 8b+8 per axis (apron clamped to L-1). */
void orc_pack_atlas(const uint8_t *dense, int32_t L, const int32_t *block_index, int64_t n_blocks,
                    uint8_t *atlas)
{
    int nb = L / 8;
    for (int64_t slot = 0; slot < (int64_t)nb * nb * nb; slot++) {
        int32_t b = block_index[slot];
        if (b < 0 || b >= n_blocks) continue;
        int bx = (int)(slot % nb), by = (int)((slot / nb) % nb), bz = (int)(slot / ((int64_t)nb * nb));
        for (int lz = 0; lz < 9; lz++)
            for (int ly = 0; ly < 9; ly++)
                for (int lx = 0; lx < 9; lx++) {
                    int gx = bx * 8 + lx, gy = by * 8 + ly, gz = bz * 8 + lz;
                    if (gx > L - 1) gx = L - 1;
                    if (gy > L - 1) gy = L - 1;
                    if (gz > L - 1) gz = L - 1;
                    const uint8_t *src = dense + (((size_t)gz * L + gy) * L + gx) * 8;
                    uint8_t *dst = atlas + (((size_t)b * 9 + lz) * 9 + ly) * 9 * 8 + (size_t)lx * 8;
                    for (int c = 0; c < 8; c++) dst[c] = src[c];
                }
    }
}

/* ---------------------------------------------------------------------------------- */
/* NEXT-2: the mip-NeRF 360 spherical contraction (Eq. 4) as a comparison   */
/* variant.  It maps lines to curves, so there is no ray-AABB skip: samples */
/* are taken at uniform contracted arc length (reading S1) by Euler steps               */
/*   t_{k+1} = t_k + Delta / sigma(t_k),  sigma = |d/dt contract(o + t d)|,             */
/* every sample is tested against the finest occupancy level, and the ray stops when    */
/* the contracted radius reaches 2 - Delta.  Canonical fp64 order (D8) as written.      */
/* ---------------------------------------------------------------------------------- */
/* contract(x) of Eq. 4: x if |x| <= 1 else (2 - 1/|x|) x/|x|.  Returns |x|. */
double orc_contract_sph(const double x[3], double c[3])
{
    double r2 = x[0] * x[0] + x[1] * x[1];
    r2 = r2 + x[2] * x[2];
    double r = sqrt(r2);
    if (r <= 1.0) { c[0] = x[0]; c[1] = x[1]; c[2] = x[2]; return r; }
    double s = 2.0 - 1.0 / r;
    for (int k = 0; k < 3; k++) { double xh = x[k] / r; c[k] = s * xh; }
    return r;
}

/* contracted speed sigma at x along unit d (derivative of Eq. 4 along the ray) */
double orc_sph_speed(const double x[3], const double d[3])
{
    double r2 = x[0] * x[0] + x[1] * x[1];
    r2 = r2 + x[2] * x[2];
    double r = sqrt(r2);
    if (r <= 1.0) return 1.0;
    double xh[3];
    for (int k = 0; k < 3; k++) xh[k] = x[k] / r;
    double dr = d[0] * xh[0] + d[1] * xh[1];
    dr = dr + d[2] * xh[2];
    double rr = r * r;
    double a = dr / rr;                          /* radial: d(2 - 1/r)/dr = 1/r^2       */
    double b = (2.0 * r - 1.0) / rr;             /* tangential: (2 - 1/r)/r             */
    double perp = 1.0 - dr * dr;
    if (perp < 0.0) perp = 0.0;
    double s2 = a * a + (b * b) * perp;
    return sqrt(s2);
}

#define ORC_SPH_MAXK(step) ((int64_t)(8.0 / (step)) + 8)

void orc_march_sph(const orc_scene *S, const double o[3], const double d[3], double t_near,
                   uint32_t flags, orc_ray_result *res, int32_t max_trace, uint64_t *trace_cells,
                   double *trace_T, int32_t *trace_count)
{
    double T = 1.0, cd[3] = {0, 0, 0}, F[4] = {0, 0, 0, 0};
    int64_t n_eval = 0, n_donly = 0, n_missing = 0;
    int32_t ntr = 0;
    int nl = S->n_levels;
    int32_t Nf = S->level_res[nl - 1];
    double t = t_near;
    const double stop = 2.0 - S->step;
    const int64_t kmax = ORC_SPH_MAXK(S->step);
    for (int64_t k = 0; k < kmax; k++) {
        double x[3], c[3];
        point_at(o, d, t, x);
        double r = orc_contract_sph(x, c);
        double cr = (r <= 1.0) ? r : (2.0 - 1.0 / r);
        if (cr >= stop) break;
        int64_t Q[3], cc[3];
        for (int a = 0; a < 3; a++) {
            Q[a] = llrint(c[a] * (double)ORC_ONE);
            cc[a] = occ_cell(Q[a], Nf);
        }
        if (get_bit(S->occ[nl - 1], (cc[2] * Nf + cc[1]) * Nf + cc[0])) {
            double tv[8];
            n_missing += orc_query_field(S, Q, tv);
            double tau = exp(tv[0]);
            double alpha = 1.0 - exp(-(tau * S->step));
            n_eval++;
            if (alpha > S->alpha_skip) {
                double w = alpha * T;
                for (int q = 0; q < 3; q++) cd[q] += w * sigmoid(tv[1 + q]);
                for (int q = 0; q < 4; q++) F[q] += w * sigmoid(tv[4 + q]);
            } else {
                n_donly++;
            }
            T = T * (1.0 - alpha);
            if (trace_cells && ntr < max_trace) {
                uint64_t cell = (uint64_t)((cc[2] * Nf + cc[1]) * Nf + cc[0]);
                trace_cells[ntr] = ((uint64_t)k << 40) | cell;
                trace_T[ntr] = T;
            }
            ntr++;
            if (!(flags & ORC_NO_EARLY_TERM) && T < S->t_min) break;
        }
        double sig = orc_sph_speed(x, d);
        t = t + S->step / sig;
    }
    double h[3];
    orc_mlp(S->mlp, cd, F, d, h);
    for (int q = 0; q < 3; q++) {
        double v = cd[q] + h[q];
        res->rgb[q] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
        res->cd[q] = cd[q];
    }
    for (int q = 0; q < 4; q++) res->F[q] = F[q];
    res->T = T;
    res->n_eval = n_eval;
    res->n_density_only = n_donly;
    res->n_skip = 0;
    res->n_missing = n_missing;
    res->n_seg = 1;
    res->region_mask = 1;
    if (trace_count) *trace_count = ntr;
}
