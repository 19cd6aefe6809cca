/*
 * ktune_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded restatement of the reference ktune executors
 * (/root/reference/proj/src/backends.cpp) used as the parity CHECKER for the
 * B200 kernels.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library; the product
 * path (paper_1802_05371_b200) never links or calls it.
 *
 * Parity is pinned: tests/test_oracle.py checks this restatement bit-for-bit
 * against the reference library itself (oracle/_ref/libktune_ref.so, built
 * from the untouched reference sources by oracle/Makefile) and against the
 * committed fixtures in tests/golden/ that were generated from it.
 *
 * The restatement is per output element rather than per tile: the tiled
 * loop nest of the reference only matters through the order in which each
 * output's products are rounded and summed, and that order is fully
 * determined by the reduction splits (k_g, k_l, k_s) -- see
 * SURVEY.md section 8(a) "A1-order":
 *
 *   c = fold_{g<k_g} ( fold_{lg<k_l} ( fold_{s<k_s} ( seq_{k in chunk(g,lg),
 *                                      (k-lo)%k_s == s} fl(a*b) ) ) )
 *
 * every fold a left fold from +0.0 with separately rounded multiply and add
 * (the reference is built without -march, so no FMA contraction happens;
 * backends.cpp:299-306 accumulate, :311-318 fold k_s sets, :320-325 merge
 * k_g slices).  Build with -ffp-contract=off to keep it that way here.
 */
#include <stdint.h>
#include <stddef.h>

#define ORACLE_API __attribute__((visibility("default")))

static int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }
static int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

/* The chunk bounds of backends.cpp:252-275: slice g of k_g over [0, K),
 * sub-slice lg of k_l inside it; empty pieces are skipped. */
typedef struct {
    int64_t lo, hi;
} span_t;

static span_t grid_slice(int64_t red, int kg, int g) {
    int64_t w = ceil_div64(red, kg);
    span_t s;
    s.lo = min64(red, (int64_t)g * w);
    s.hi = min64(red, s.lo + w);
    return s;
}

static span_t group_slice(span_t slice, int kl, int lg) {
    int64_t w = ceil_div64(slice.hi - slice.lo, kl);
    span_t s;
    s.lo = min64(slice.hi, slice.lo + (int64_t)lg * w);
    s.hi = min64(slice.hi, s.lo + w);
    return s;
}

/* ------------------------------------------------------------------------ */
/* GEMM: backends.cpp:228-329.  A is M x K (K x M when ta), B is K x N       */
/* (N x K when tb), C is M x N row-major.  tuning = {m_s,n_s,m_l,n_l,u,k_s,  */
/* k_l,k_g}; only the three reduction splits affect the result.              */
/* ------------------------------------------------------------------------ */

#define DEFINE_GEMM(NAME, T)                                                   \
    ORACLE_API void NAME(int64_t M, int64_t N, int64_t K, int ta, int tb,     \
                         const int32_t* tuning, const T* a, const T* b, T* c) \
    {                                                                          \
        const int ks = tuning[5], kl = tuning[6], kg = tuning[7];              \
        for (int64_t i = 0; i < M; ++i) {                                      \
            for (int64_t j = 0; j < N; ++j) {                                  \
                T out = (T)0;                                                  \
                for (int g = 0; g < kg; ++g) {                                 \
                    span_t sl = grid_slice(K, kg, g);                          \
                    if (sl.lo >= sl.hi) continue;                              \
                    T blk = (T)0;                                              \
                    for (int lg = 0; lg < kl; ++lg) {                          \
                        span_t gr = group_slice(sl, kl, lg);                   \
                        if (gr.lo >= gr.hi) continue;                          \
                        for (int s = 0; s < ks; ++s) {                         \
                            T acc = (T)0;                                      \
                            for (int64_t k = gr.lo + s; k < gr.hi; k += ks) {  \
                                T av = ta ? a[k * M + i] : a[i * K + k];       \
                                T bv = tb ? b[j * K + k] : b[k * N + j];       \
                                T prod = av * bv;                              \
                                acc = acc + prod;                              \
                            }                                                  \
                            blk = blk + acc;                                   \
                        }                                                      \
                    }                                                          \
                    out = out + blk;                                           \
                }                                                              \
                c[i * N + j] = out;                                            \
            }                                                                  \
        }                                                                      \
    }

DEFINE_GEMM(oracle_execute_gemm_f32, float)
DEFINE_GEMM(oracle_execute_gemm_f64, double)

/* ------------------------------------------------------------------------ */
/* CONV (valid mode): backends.cpp:331-444 with the indirection table of    */
/* backends.cpp:197-216.  images C,H,W,N; filters C,R,S,K; outputs K,P,Q,N. */
/* dims = {n,p,q,k,c,r,s}; tuning = {k_s,p_s,q_s,n_s,k_l,p_l,q_l,n_l,u,c_s, */
/* c_l,c_g}; only c_s, c_l, c_g affect the result.                           */
/* ------------------------------------------------------------------------ */

ORACLE_API void oracle_indirection_table(const int64_t* dims, int64_t* out4)
{
    const int64_t Nb = dims[0], P = dims[1], Q = dims[2], C = dims[4],
                  R = dims[5], S = dims[6];
    const int64_t W = Q + S - 1, H = P + R - 1;
    int64_t t = 0;
    for (int64_t c = 0; c < C; ++c)
        for (int64_t r = 0; r < R; ++r)
            for (int64_t s = 0; s < S; ++s, ++t) {
                out4[4 * t + 0] = c;
                out4[4 * t + 1] = r;
                out4[4 * t + 2] = s;
                out4[4 * t + 3] = c * H * W * Nb + r * W * Nb + s * Nb;
            }
}

#define DEFINE_CONV(NAME, T)                                                   \
    ORACLE_API void NAME(const int64_t* dims, const int32_t* tuning,           \
                         const T* img, const T* flt, T* out)                   \
    {                                                                          \
        const int64_t Nb = dims[0], P = dims[1], Q = dims[2], K = dims[3],    \
                      C = dims[4], R = dims[5], S = dims[6];                   \
        const int64_t H = P + R - 1, W = Q + S - 1, CRS = C * R * S;          \
        const int cs = tuning[9], cl = tuning[10], cg = tuning[11];            \
        for (int64_t k = 0; k < K; ++k)                                        \
        for (int64_t p = 0; p < P; ++p)                                        \
        for (int64_t q = 0; q < Q; ++q)                                        \
        for (int64_t n = 0; n < Nb; ++n) {                                     \
            const int64_t base = (p * W + q) * Nb + n;                         \
            T o = (T)0;                                                        \
            for (int g = 0; g < cg; ++g) {                                     \
                span_t sl = grid_slice(CRS, cg, g);                            \
                if (sl.lo >= sl.hi) continue;                                  \
                T blk = (T)0;                                                  \
                for (int lg = 0; lg < cl; ++lg) {                              \
                    span_t gr = group_slice(sl, cl, lg);                       \
                    if (gr.lo >= gr.hi) continue;                              \
                    for (int s = 0; s < cs; ++s) {                             \
                        T acc = (T)0;                                          \
                        for (int64_t t = gr.lo + s; t < gr.hi; t += cs) {      \
                            const int64_t ci = t / (R * S);                    \
                            const int64_t ri = (t / S) % R;                    \
                            const int64_t si = t % S;                          \
                            const int64_t off = ci * H * W * Nb +              \
                                                ri * W * Nb + si * Nb;         \
                            T fv = flt[t * K + k];                             \
                            T iv = img[base + off];                            \
                            T prod = fv * iv;                                  \
                            acc = acc + prod;                                  \
                        }                                                      \
                        blk = blk + acc;                                       \
                    }                                                          \
                }                                                              \
                o = o + blk;                                                   \
            }                                                                  \
            out[((k * P + p) * Q + q) * Nb + n] = o;                           \
        }                                                                      \
    }

DEFINE_CONV(oracle_execute_conv_f32, float)
DEFINE_CONV(oracle_execute_conv_f64, double)

/* ------------------------------------------------------------------------ */
/* Tuning-independent references of the reference's own tests:              */
/* naive double-accumulated GEMM (test_backends.cpp:17-34) and the direct   */
/* seven-loop convolution (test_backends.cpp:38-66).  Used for the fast-mode */
/* and tensor-core tolerances (metric max|got-ref|/max(|ref|,1),            */
/* test_backends.cpp:74-82).  Outputs are double (no final rounding) so the */
/* caller can compare against any output precision.                          */
/* ------------------------------------------------------------------------ */

#define DEFINE_NAIVE_GEMM(NAME, T)                                             \
    ORACLE_API void NAME(int64_t M, int64_t N, int64_t K, int ta, int tb,     \
                         const T* a, const T* b, double* c)                    \
    {                                                                          \
        for (int64_t i = 0; i < M; ++i)                                        \
            for (int64_t j = 0; j < N; ++j) {                                  \
                double acc = 0.0;                                              \
                for (int64_t k = 0; k < K; ++k) {                              \
                    double av = ta ? a[k * M + i] : a[i * K + k];              \
                    double bv = tb ? b[j * K + k] : b[k * N + j];              \
                    acc += av * bv;                                            \
                }                                                              \
                c[i * N + j] = acc;                                            \
            }                                                                  \
    }

DEFINE_NAIVE_GEMM(oracle_naive_gemm_f32, float)
DEFINE_NAIVE_GEMM(oracle_naive_gemm_f64, double)

#define DEFINE_DIRECT_CONV(NAME, T)                                            \
    ORACLE_API void NAME(const int64_t* dims, const T* img, const T* flt,      \
                         double* out)                                          \
    {                                                                          \
        const int64_t Nb = dims[0], P = dims[1], Q = dims[2], K = dims[3],    \
                      C = dims[4], R = dims[5], S = dims[6];                   \
        const int64_t H = P + R - 1, W = Q + S - 1;                            \
        for (int64_t k = 0; k < K; ++k)                                        \
        for (int64_t p = 0; p < P; ++p)                                        \
        for (int64_t q = 0; q < Q; ++q)                                        \
        for (int64_t n = 0; n < Nb; ++n) {                                     \
            double acc = 0.0;                                                  \
            for (int64_t c = 0; c < C; ++c)                                    \
            for (int64_t r = 0; r < R; ++r)                                    \
            for (int64_t s = 0; s < S; ++s) {                                  \
                double iv = img[((c * H + p + r) * W + q + s) * Nb + n];       \
                double fv = flt[((c * R + r) * S + s) * K + k];                \
                acc += iv * fv;                                                \
            }                                                                  \
            out[((k * P + p) * Q + q) * Nb + n] = acc;                         \
        }                                                                      \
    }

DEFINE_DIRECT_CONV(oracle_direct_conv_f32, float)
DEFINE_DIRECT_CONV(oracle_direct_conv_f64, double)

/* Seeded operand fill of CpuBackend::measure (backends.cpp:481-484, 508-513)
 * and of the reference tests (test_backends.cpp:68-71): std::mt19937_64 with
 * unit_real = (rng() >> 11) * 2^-53 (sampler.cpp:14-17).  A self-contained
 * MT19937-64 so the checker does not depend on libstdc++. */
typedef struct {
    uint64_t mt[312];
    int mti;
} mt64_t;

static void mt64_seed(mt64_t* s, uint64_t seed)
{
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->mti = 312;
}

static uint64_t mt64_next(mt64_t* s)
{
    static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    if (s->mti >= 312) {
        int i;
        for (i = 0; i < 312 - 156; ++i) {
            uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[i + 1] & 0x7FFFFFFFULL);
            s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        for (; i < 311; ++i) {
            uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[i + 1] & 0x7FFFFFFFULL);
            s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        uint64_t x = (s->mt[311] & 0xFFFFFFFF80000000ULL) | (s->mt[0] & 0x7FFFFFFFULL);
        s->mt[311] = s->mt[155] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        s->mti = 0;
    }
    uint64_t x = s->mt[s->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* Fills n values from one engine: lo=0 → unit_real in [0,1) (harness fill);
 * lo=-1 → 2*unit_real-1 in [-1,1) (test fill).  Two buffers drawn in
 * sequence from the same seed match "fill a, then fill b". */
ORACLE_API void oracle_fill_f32(uint64_t seed, int symmetric, float* a, int64_t na,
                                float* b, int64_t nb)
{
    mt64_t s;
    mt64_seed(&s, seed);
    for (int64_t i = 0; i < na; ++i) {
        double u = (double)(mt64_next(&s) >> 11) * 0x1.0p-53;
        a[i] = (float)(symmetric ? 2.0 * u - 1.0 : u);
    }
    for (int64_t i = 0; i < nb; ++i) {
        double u = (double)(mt64_next(&s) >> 11) * 0x1.0p-53;
        b[i] = (float)(symmetric ? 2.0 * u - 1.0 : u);
    }
}

ORACLE_API void oracle_fill_f64(uint64_t seed, int symmetric, double* a, int64_t na,
                                double* b, int64_t nb)
{
    mt64_t s;
    mt64_seed(&s, seed);
    for (int64_t i = 0; i < na; ++i) {
        double u = (double)(mt64_next(&s) >> 11) * 0x1.0p-53;
        a[i] = symmetric ? 2.0 * u - 1.0 : u;
    }
    for (int64_t i = 0; i < nb; ++i) {
        double u = (double)(mt64_next(&s) >> 11) * 0x1.0p-53;
        b[i] = symmetric ? 2.0 * u - 1.0 : u;
    }
}
