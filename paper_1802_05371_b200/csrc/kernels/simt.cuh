// simt.cuh -- K1/K2/K3: the fp32/fp64 SIMT family for sm_100a.
//
// One kernel body serves GEMM (backends.cpp:228-329) and implicit-GEMM CONV
// (backends.cpp:331-444): both are "rows x cols += A[rows, red] * B[red, cols]"
// over a reduction axis (GEMM K, CONV C*R*S), differing only in address
// generation, which a Problem policy supplies.
//
// Mapping of the ISAAC tuple (param_space.hpp:52-63):
//   m_l x n_l  block output tile          (grid x = column tiles, y = row tiles)
//   m_s x n_s  per-thread register tile   (template MS, NS; strided ownership:
//              thread (ty,tx) owns rows ty+i*tm and cols tx+j*tn, so smem reads
//              are conflict-free and stores coalesce)
//   k_l        thread groups per block, each owning one contiguous sub-range
//              of the block's reduction slice; their partial tiles are folded
//              through shared memory in group order
//   k_s        interleaved accumulator sets inside a thread (template KS)
//   u          reduction depth staged per step (cp.async, double-buffered);
//              each group stages w = max(u/k_l, k_s) columns per step so the
//              block's staging footprint equals the resource model
//              2*size*(m_l*u + u*n_l) of param_space.cpp:209-210
//   k_g        grid slices (grid z); slices 0..nz-2 publish partial tiles
//              to a workspace, the last slice's block folds them in slice
//              order (single launch, no memset, deterministic: the "merge
//              pass" of backends.cpp:90-112 fused into the main kernel)
//
// PARITY mode reproduces the reference summation order bit-for-bit
// (separately rounded __fmul_rn/__fadd_rn, left folds from +0.0 in the order
// spelled out in oracle/ktune_oracle.c).  FAST mode uses FFMA with the same
// structure (|err| <= 1e-5 relative, test_backends.cpp:142).

#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ktune_dev {

struct SimtParams {
    std::int64_t rows;      // GEMM M, CONV K filters
    std::int64_t red;       // GEMM K, CONV C*R*S
    std::int64_t out_elems; // size of the output (workspace slice stride)
    int ml, nl;             // block tile (nl = p_l*q_l*n_l for CONV)
    int ms, ns, ks;         // runtime copies of the register tile (generic kernel)
    int kl;                 // groups
    int tm, tn;             // threads per group along rows / cols
    int w;                  // staged reduction columns per group per step
    int pad_a, pad_b;       // smem row pads
    std::int64_t kg_span;   // ceil(red / k_g)
    int nz;                 // non-empty grid slices (= gridDim.z)
    void* out;              // C / outputs
    void* ws;               // k_g partials [nz-1][out_elems]
    unsigned long long* flags;  // [nz-1][tiles] publication tokens
    unsigned long long token;   // unique per launch (never 0)
};

// ---- GEMM policy: A is M x K (K x M when ta), B is K x N (N x K when tb) ----
template <typename T>
struct GemmProblem {
    const T* a;
    const T* b;
    std::int64_t M, N, K;
    int ta, tb;
    int nl;
    // A tile loads are contiguous along the reduction axis unless transposed.
    __device__ bool a_red_contig() const { return !ta; }
    __device__ bool b_red_contig() const { return tb; }
    __device__ const T* a_addr(std::int64_t row, std::int64_t t) const {
        return ta ? a + t * M + row : a + row * K + t;
    }
    // column "base" = global column index j
    __device__ const T* b_addr(std::int64_t t, std::int64_t base) const {
        return tb ? b + base * K + t : b + t * N + base;
    }
    // base and output offset of local column x of column tile ct; -1 if outside.
    __device__ void column(int ct, int x, std::int64_t& base, std::int64_t& out_col) const {
        const std::int64_t j = std::int64_t(ct) * nl + x;
        base = j < N ? j : -1;
        out_col = base;
    }
    __device__ std::int64_t out_index(std::int64_t row, std::int64_t out_col) const { return row * N + out_col; }
};

// ---- CONV policy: images C,H,W,N; filters C,R,S,K; outputs K,P,Q,N --------
// A = filters viewed as CRS x K (row = filter k, contiguous along k);
// B = the image gather: column (p,q,n) reads images[(p*W+q)*N + n + off(t)]
// with off(t) the indirection-table offset of backends.cpp:197-216.
template <typename T>
struct ConvProblem {
    const T* flt;
    const T* img;
    std::int64_t Nb, P, Q, K, C, R, S, H, W;
    int pl, ql, nlb;              // spatial block tile
    int tiles_q, tiles_n;         // column-tile grid decomposition
    __device__ bool a_red_contig() const { return false; }
    __device__ bool b_red_contig() const { return false; }
    __device__ const T* a_addr(std::int64_t row, std::int64_t t) const { return flt + t * K + row; }
    __device__ std::int64_t off(std::int64_t t) const {
        const std::int64_t rs = R * S;
        const std::int64_t c = t / rs;
        const std::int64_t rem = t - c * rs;
        const std::int64_t r = rem / S;
        const std::int64_t s = rem - r * S;
        return (c * H + r) * W * Nb + s * Nb;
    }
    __device__ const T* b_addr(std::int64_t t, std::int64_t base) const { return img + base + off(t); }
    __device__ void column(int ct, int x, std::int64_t& base, std::int64_t& out_col) const {
        const int tn_ = ct % tiles_n;
        const int rest = ct / tiles_n;
        const int tq = rest % tiles_q;
        const int tp = rest / tiles_q;
        const int nn = x % nlb;
        const int qq = (x / nlb) % ql;
        const int pp = x / (nlb * ql);
        const std::int64_t p = std::int64_t(tp) * pl + pp, q = std::int64_t(tq) * ql + qq,
                           n = std::int64_t(tn_) * nlb + nn;
        if (p < P && q < Q && n < Nb) {
            base = (p * W + q) * Nb + n;
            out_col = (p * Q + q) * Nb + n;
        } else {
            base = -1;
            out_col = -1;
        }
    }
    __device__ std::int64_t out_index(std::int64_t row, std::int64_t out_col) const {
        return row * (P * Q * Nb) + out_col;
    }
};

// ---- arithmetic of the two modes ------------------------------------------
template <typename T, bool PARITY>
struct Arith;

template <>
struct Arith<float, true> {
    static __device__ __forceinline__ float mac(float acc, float a, float b) { return __fadd_rn(acc, __fmul_rn(a, b)); }
    static __device__ __forceinline__ float add(float x, float y) { return __fadd_rn(x, y); }
};
template <>
struct Arith<float, false> {
    static __device__ __forceinline__ float mac(float acc, float a, float b) { return fmaf(a, b, acc); }
    static __device__ __forceinline__ float add(float x, float y) { return __fadd_rn(x, y); }
};
template <>
struct Arith<double, true> {
    static __device__ __forceinline__ double mac(double acc, double a, double b) {
        return __dadd_rn(acc, __dmul_rn(a, b));
    }
    static __device__ __forceinline__ double add(double x, double y) { return __dadd_rn(x, y); }
};
template <>
struct Arith<double, false> {
    static __device__ __forceinline__ double mac(double acc, double a, double b) { return fma(a, b, acc); }
    static __device__ __forceinline__ double add(double x, double y) { return __dadd_rn(x, y); }
};

// ---- cp.async (LDGSTS) with zero-fill for out-of-range elements ------------
template <int BYTES>
__device__ __forceinline__ void cp_async_zfill(void* smem, const void* gmem, bool valid) {
    const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int src_bytes = valid ? BYTES : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(saddr), "l"(gmem), "n"(BYTES),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Generic (runtime-tile) kernels keep accumulators in local memory up to this
// many per thread; larger register tiles are rejected at launch.
constexpr int kGenericMaxAcc = 256;

template <int MS, int NS, int KS>
struct LaunchCap {
    // Keep the register budget honest: big register tiles only with few threads.
    static constexpr int acc = (MS == 0) ? kGenericMaxAcc : MS * NS * KS;
    static constexpr int threads = (MS == 0) ? 1024 : (acc <= 16 ? 1024 : (acc <= 64 ? 512 : 256));
};

template <class Prob, typename T, int MS_, int NS_, int KS_, bool PARITY>
__global__ void __launch_bounds__(LaunchCap<MS_, NS_, KS_>::threads)
    simt_kernel(const Prob prob, const SimtParams p) {
    constexpr bool RT = (MS_ == 0);  // runtime-tile generic kernel
    const int MS = RT ? p.ms : MS_;
    const int NS = RT ? p.ns : NS_;
    const int KS = RT ? p.ks : KS_;
    constexpr int ACC = RT ? kGenericMaxAcc : (MS_ * NS_ * KS_);
    constexpr int TILE = RT ? kGenericMaxAcc : (MS_ * NS_);
    using A = Arith<T, PARITY>;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    // smem: [col_base nl i64][col_out nl i64][As 2 x kl x w x (ml+pad_a)][Bs 2 x kl x w x (nl+pad_b)]
    std::int64_t* col_base = reinterpret_cast<std::int64_t*>(smem_raw);
    std::int64_t* col_out = col_base + p.nl;
    T* As = reinterpret_cast<T*>(col_out + p.nl);
    const int a_ld = p.ml + p.pad_a, b_ld = p.nl + p.pad_b;
    const int a_group = p.w * a_ld, b_group = p.w * b_ld;
    T* Bs = As + 2 * p.kl * a_group;

    const int tid = threadIdx.x;
    const int nthreads = blockDim.x;
    const int per_group = p.tm * p.tn;
    const int lg = tid / per_group;
    const int r_in = tid - lg * per_group;
    const int ty = r_in / p.tn;
    const int tx = r_in - ty * p.tn;
    const int ct = blockIdx.x, rt = blockIdx.y, g = blockIdx.z;
    const std::int64_t row0 = std::int64_t(rt) * p.ml;

    // Grid slice g and the k_l sub-ranges inside it (backends.cpp:252-275).
    const std::int64_t s_lo = min(p.red, std::int64_t(g) * p.kg_span);
    const std::int64_t s_hi = min(p.red, s_lo + p.kg_span);
    const std::int64_t kl_span = (s_hi - s_lo + p.kl - 1) / p.kl;
    const std::int64_t nsteps = (kl_span + p.w - 1) / p.w;

    for (int x = tid; x < p.nl; x += nthreads) prob.column(ct, x, col_base[x], col_out[x]);
    __syncthreads();

    // Stage step `st` for every group into buffer `buf`.
    auto stage = [&](std::int64_t st, int buf) {
        const int a_elems = p.kl * p.w * p.ml;
        const bool a_rc = prob.a_red_contig();
        for (int e = tid; e < a_elems; e += nthreads) {
            const int gx = e / (p.w * p.ml);
            const int rem = e - gx * (p.w * p.ml);
            int kk, ii;
            if (a_rc) { ii = rem / p.w; kk = rem - ii * p.w; }
            else      { kk = rem / p.ml; ii = rem - kk * p.ml; }
            const std::int64_t glo = min(s_hi, s_lo + gx * kl_span);
            const std::int64_t ghi = min(s_hi, glo + kl_span);
            const std::int64_t t = glo + st * p.w + kk;
            const std::int64_t row = row0 + ii;
            const bool ok = (t < ghi) && (row < p.rows);
            const T* src = ok ? prob.a_addr(row, t) : reinterpret_cast<const T*>(p.out);
            cp_async_zfill<sizeof(T)>(As + (buf * p.kl + gx) * a_group + kk * a_ld + ii, src, ok);
        }
        const int b_elems = p.kl * p.w * p.nl;
        const bool b_rc = prob.b_red_contig();
        for (int e = tid; e < b_elems; e += nthreads) {
            const int gx = e / (p.w * p.nl);
            const int rem = e - gx * (p.w * p.nl);
            int kk, xx;
            if (b_rc) { xx = rem / p.w; kk = rem - xx * p.w; }
            else      { kk = rem / p.nl; xx = rem - kk * p.nl; }
            const std::int64_t glo = min(s_hi, s_lo + gx * kl_span);
            const std::int64_t ghi = min(s_hi, glo + kl_span);
            const std::int64_t t = glo + st * p.w + kk;
            const std::int64_t base = col_base[xx];
            const bool ok = (t < ghi) && (base >= 0);
            const T* src = ok ? prob.b_addr(t, base) : reinterpret_cast<const T*>(p.out);
            cp_async_zfill<sizeof(T)>(Bs + (buf * p.kl + gx) * b_group + kk * b_ld + xx, src, ok);
        }
        cp_async_commit();
    };

    T acc[ACC];
#pragma unroll
    for (int i = 0; i < ACC; ++i) acc[i] = T(0);

    const std::int64_t my_lo = min(s_hi, s_lo + lg * kl_span);
    const std::int64_t my_hi = min(s_hi, my_lo + kl_span);

    if (nsteps > 0) stage(0, 0);
    for (std::int64_t st = 0; st < nsteps; ++st) {
        const int buf = int(st & 1);
        if (st + 1 < nsteps) {
            stage(st + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const std::int64_t k0 = my_lo + st * p.w;
        const int nv = int(max(std::int64_t(0), min(std::int64_t(p.w), my_hi - k0)));
        const T* as = As + (buf * p.kl + lg) * a_group;
        const T* bs = Bs + (buf * p.kl + lg) * b_group;
        for (int kk0 = 0; kk0 < nv; kk0 += KS) {
#pragma unroll
            for (int s = 0; s < (RT ? 1 : KS_); ++s) {
                // generic kernel: iterate sets at runtime
                for (int sr = 0; sr < (RT ? KS : 1); ++sr) {
                    const int set = RT ? sr : s;
                    const int kk = kk0 + set;
                    if (kk < nv) {
                        T av[RT ? 16 : (MS_ > 0 ? MS_ : 1)];
                        T bv[RT ? 16 : (NS_ > 0 ? NS_ : 1)];
                        if constexpr (RT) {
                            // runtime tiles read operands on the fly
                            for (int i = 0; i < MS; ++i) {
                                const T a_ = as[kk * a_ld + ty + i * p.tm];
                                for (int j = 0; j < NS; ++j) {
                                    const T b_ = bs[kk * b_ld + tx + j * p.tn];
                                    T& c_ = acc[(set * MS + i) * NS + j];
                                    c_ = A::mac(c_, a_, b_);
                                }
                            }
                            (void)av;
                            (void)bv;
                        } else {
#pragma unroll
                            for (int i = 0; i < MS_; ++i) av[i] = as[kk * a_ld + ty + i * p.tm];
#pragma unroll
                            for (int j = 0; j < NS_; ++j) bv[j] = bs[kk * b_ld + tx + j * p.tn];
#pragma unroll
                            for (int i = 0; i < MS_; ++i)
#pragma unroll
                                for (int j = 0; j < NS_; ++j) {
                                    T& c_ = acc[(set * MS_ + i) * NS_ + j];
                                    c_ = A::mac(c_, av[i], bv[j]);
                                }
                        }
                    }
                }
            }
        }
        __syncthreads();
    }

    // ---- fold: k_s sets within a thread, then k_l groups in order ----------
    // (backends.cpp:311-318): blk = ((0 + g0s0) + g0s1) + ... + g1s0 + ...
    T blk[TILE];
    T* red = As;  // reuse operand smem as an m_l x n_l tile
    const int red_ld = p.nl;
    const bool my_nonempty = my_lo < my_hi;
    for (int step = 0; step < p.kl; ++step) {
        if (lg == step) {
#pragma unroll
            for (int i = 0; i < MS; ++i)
#pragma unroll
                for (int j = 0; j < NS; ++j) {
                    T v = (step == 0) ? T(0) : red[(ty + i * p.tm) * red_ld + tx + j * p.tn];
                    if (my_nonempty)
#pragma unroll
                        for (int s = 0; s < KS; ++s) v = A::add(v, acc[(s * MS + i) * NS + j]);
                    blk[i * NS + j] = v;
                    if (step + 1 < p.kl) red[(ty + i * p.tm) * red_ld + tx + j * p.tn] = v;
                }
        }
        __syncthreads();
    }

    // ---- output: direct store, or k_g partial + last-block ordered merge ---
    const bool owner = (lg == p.kl - 1);
    T* out = static_cast<T*>(p.out);
    if (p.nz == 1) {
        if (owner)
#pragma unroll
            for (int i = 0; i < MS; ++i) {
                const std::int64_t row = row0 + ty + i * p.tm;
                if (row >= p.rows) continue;
                for (int j = 0; j < NS; ++j) {
                    const std::int64_t oc = col_out[tx + j * p.tn];
                    if (oc >= 0) out[prob.out_index(row, oc)] = A::add(T(0), blk[i * NS + j]);
                }
            }
        return;
    }
    // Slices 0..nz-2 publish their partial tile and a per-launch token; the
    // block of the last slice (scheduled after every lower-z block has
    // started, so the wait cannot deadlock) waits for all tokens and folds
    // the partials in slice order, its own last (backends.cpp:320-325).
    // Tokens are unique per launch, so the workspace never needs zeroing.
    T* ws = static_cast<T*>(p.ws);
    const std::int64_t tiles = std::int64_t(gridDim.x) * gridDim.y;
    const std::int64_t tile_id = std::int64_t(rt) * gridDim.x + ct;
    if (g < p.nz - 1) {
        if (owner)
#pragma unroll
            for (int i = 0; i < MS; ++i) {
                const std::int64_t row = row0 + ty + i * p.tm;
                if (row >= p.rows) continue;
#pragma unroll
                for (int j = 0; j < NS; ++j) {
                    const std::int64_t oc = col_out[tx + j * p.tn];
                    if (oc >= 0) __stcg(ws + std::int64_t(g) * p.out_elems + prob.out_index(row, oc), blk[i * NS + j]);
                }
            }
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            unsigned long long* flag = p.flags + std::int64_t(g) * tiles + tile_id;
            asm volatile("st.release.gpu.global.u64 [%0], %1;\n" ::"l"(flag), "l"(p.token) : "memory");
        }
        return;
    }
    if (tid == 0) {
        for (int gg = 0; gg < p.nz - 1; ++gg) {
            const unsigned long long* flag = p.flags + std::int64_t(gg) * tiles + tile_id;
            unsigned long long v;
            while (true) {
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(flag) : "memory");
                if (v == p.token) break;
                __nanosleep(64);
            }
        }
    }
    __syncthreads();
    if (owner)
#pragma unroll
        for (int i = 0; i < MS; ++i) {
            const std::int64_t row = row0 + ty + i * p.tm;
            if (row >= p.rows) continue;
#pragma unroll
            for (int j = 0; j < NS; ++j) {
                const std::int64_t oc = col_out[tx + j * p.tn];
                if (oc < 0) continue;
                const std::int64_t idx = prob.out_index(row, oc);
                T v = T(0);
                for (int gg = 0; gg < p.nz - 1; ++gg)
                    v = A::add(v, __ldcg(ws + std::int64_t(gg) * p.out_elems + idx));
                out[idx] = A::add(v, blk[i * NS + j]);
            }
        }
}

}  // namespace ktune_dev
