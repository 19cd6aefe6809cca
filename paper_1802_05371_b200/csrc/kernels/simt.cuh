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
#include <type_traits>
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
    int lw, lml, lnl;       // log2 of w, ml, nl (all powers of two)
    int lva, lvb;           // log2 of the cp.async vector width (elements) of A / B
    int a_ld, b_ld;         // smem leading dimension of the A / B tiles
    int a_group, b_group;   // elements of one group's A / B tile (incl. padding)
    int a_stage, b_stage;   // elements of one pipeline stage (all groups)
    int stages;             // cp.async pipeline depth (2..8)
    std::int64_t kg_span;   // ceil(red / k_g)
    int nz;                 // non-empty grid slices (= gridDim.z)
    void* out;              // C / outputs
    void* ws;               // k_g partials [nz-1][out_elems]
    unsigned long long* flags;  // [nz-1][tiles] publication tokens
    unsigned long long token;   // unique per launch (never 0)
    int fast_ld;                // affine problems: per-thread chunk state precomputed (see ChunkLd)
    int gather_ld;              // CONV: per-thread gather chunk state precomputed (see GatherLd)
    long long* dbg;             // optional timeline probe (KTUNE_SIMT_DEBUG): blocks x = 0, y in {0, 1}
    void* acc;                  // FAST k_g merge by reduction: zeroed [out_elems] accumulator, or nullptr
};

// Timeline probe (debug builds of a measurement: KTUNE_SIMT_DEBUG = device
// address of a [blocks][8] int64 buffer): thread 0 of every block records
// %globaltimer at up to 8 points, plus its SM id in slot 7.
__device__ __forceinline__ void simt_probe(const SimtParams& p, int slot) {
    if (p.dbg == nullptr || threadIdx.x != 0) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const std::int64_t b = (std::int64_t(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    p.dbg[b * 8 + slot] = (long long)t;
    if (slot == 0) {
        unsigned sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        p.dbg[b * 8 + 7] = sm;
    }
}

// Per-thread cp.async chunks of one operand, precomputed once per block for
// problems whose addresses are affine in the reduction index (GEMM): element
// offset at the block's first step, smem destination, remaining reduction
// columns and valid lanes.  A step then costs a few integer ops per chunk
// instead of the full index decomposition.
constexpr int kChunkMax = 4;
struct ChunkLd {
    int off;  // element offset of the chunk at step 0 (operand < 2^31 elements)
    int dst;  // element offset inside one stage
    int lim;  // reduction columns left in the group from the chunk's first column
    int cnt;  // valid elements along the contiguous dimension (0 = chunk outside the tensor)
};

// ---- GEMM policy: A is M x K (K x M when ta), B is K x N (N x K when tb) ----
template <typename T>
struct GemmProblem {
    static constexpr bool kAffine = true;   // both operands affine in the reduction index
    static constexpr bool kAffineA = true;
    const T* a;
    const T* b;
    std::int64_t M, N, K;
    int ta, tb;
    int nl;
    // Valid leading elements of a v-chunk of B columns starting at `base`
    // (columns are contiguous global indices).
    __device__ int b_cols_valid(std::int64_t base, int v) const {
        return base < 0 ? 0 : int(min(std::int64_t(v), N - base));
    }
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
    // element distance of one reduction step along each operand
    __device__ std::int64_t a_kstride() const { return ta ? M : 1; }
    __device__ std::int64_t b_kstride() const { return tb ? 1 : N; }
};

// ---- CONV policy: images C,H,W,N; filters C,R,S,K; outputs K,P,Q,N --------
// A = filters viewed as CRS x K (row = filter k, contiguous along k);
// B = the image gather: column (p,q,n) reads images[(p*W+q)*N + n + off(t)]
// with off(t) the indirection-table offset of backends.cpp:197-216.
template <typename T>
struct ConvProblem {
    static constexpr bool kAffine = false;  // the image gather is not (tap decomposition)
    static constexpr bool kAffineA = true;  // the filters are: flt + t*K + row
    const T* flt;
    const T* img;
    std::int64_t Nb, P, Q, K, C, R, S, H, W;
    int pl, ql, nlb;              // spatial block tile
    int tiles_q, tiles_n;         // column-tile grid decomposition
    std::int64_t hwn, wn;         // image strides of a channel and of a row
    // t / (R*S) and rem / S as multiply-high by ceil(2^32 / d) (exact while
    // t * R*S < 2^32, host-checked; magic = 0 keeps the divisions); d = 1
    // has no 32-bit multiplier and passes n through the mask instead
    unsigned magic, m_rs, m_s, one_rs, one_s;
    // The host only vectorises the gather when n-runs are whole chunks, so a
    // chunk is entirely valid or entirely outside the tensor.
    __device__ int b_cols_valid(std::int64_t base, int v) const { return base < 0 ? 0 : v; }
    __device__ const T* a_addr(std::int64_t row, std::int64_t t) const { return flt + t * K + row; }
    __device__ std::int64_t a_kstride() const { return K; }
    // t = (c*R + r)*S + s -> image offset of the tap (the indirection table
    // entry of backends.cpp:197-216).  The reduction index fits in 32 bits
    // (host-checked), so the decomposition uses 32-bit divisions: the 64-bit
    // ones dominated the gather loader's instruction count.
    __device__ std::int64_t off(std::int64_t t) const {
        const unsigned tt = unsigned(t), rs = unsigned(R * S), ss = unsigned(S);
        unsigned c, r;
        if (magic) {
            c = __umulhi(tt, m_rs) + (tt & one_rs);
        } else {
            c = tt / rs;
        }
        const unsigned rem = tt - c * rs;
        if (magic) {
            r = __umulhi(rem, m_s) + (rem & one_s);
        } else {
            r = rem / ss;
        }
        const unsigned s = rem - r * ss;
        return std::int64_t(c) * hwn + std::int64_t(r) * wn + std::int64_t(s) * Nb;
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

// ---- programmatic dependent launch ----------------------------------------
// Launched with programmatic stream serialization, a kernel lets the next
// one on its stream start its prologue as soon as every block of this one is
// running; the next kernel's global-memory work waits for this one's
// completion in pdl_wait().  Without the attribute both are no-ops.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

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
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
// Copies the first src_bytes of a BYTES chunk and zero-fills the rest (an
// invalid chunk has src_bytes 0 and reads nothing).
template <int BYTES>
__device__ __forceinline__ void cp_async_zfill(void* smem, const void* gmem, int src_bytes) {
    const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    if constexpr (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem), "r"(src_bytes));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(saddr), "l"(gmem), "n"(BYTES),
                     "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_wait_dyn(int n) {
    switch (n) {
        case 0: cp_async_wait<0>(); break;
        case 1: cp_async_wait<1>(); break;
        case 2: cp_async_wait<2>(); break;
        case 3: cp_async_wait<3>(); break;
        case 4: cp_async_wait<4>(); break;
        case 5: cp_async_wait<5>(); break;
        default: cp_async_wait<6>(); break;
    }
}

// ---- output: direct store, or the k_g merge by the last-arriving slice ----
// Every slice publishes its partial tile to ws[g] and takes a ticket from the
// tile's 32-bit arrival counter (one acq_rel atomic add).  The slice that
// arrives last -- whichever z it has -- folds all partials in slice order,
// its own from registers (backends.cpp:320-325: c = ((0 + s_0) + s_1) + ...)
// and resets the counter to zero for the next launch on this workspace.  No
// block ever waits for another, so nothing depends on the order blocks are
// dispatched in.  Must be reached by every thread of the block.
template <typename T, bool PARITY, int TILE, class Prob, class IdxFn>
__device__ __forceinline__ void simt_store_or_merge(const Prob& prob, const SimtParams& p, const T* blk, int n,
                                                    bool owner, IdxFn idx_of) {
    using A = Arith<T, PARITY>;
    T* out = static_cast<T*>(p.out);
    if (p.nz == 1) {
        if (owner)
#pragma unroll
            for (int e = 0; e < TILE; ++e) {
                if (e >= n) break;
                std::int64_t row, oc;
                idx_of(e, row, oc);
                if (row < p.rows && oc >= 0) out[prob.out_index(row, oc)] = A::add(T(0), blk[e]);
            }
        return;
    }
    T* ws = static_cast<T*>(p.ws);
    const int g = int(blockIdx.z);
    const std::int64_t tile_id = std::int64_t(blockIdx.y) * gridDim.x + blockIdx.x;
    std::int64_t idx[TILE];
#pragma unroll
    for (int e = 0; e < TILE; ++e) {
        idx[e] = -1;
        if (e < n) {
            std::int64_t row, oc;
            idx_of(e, row, oc);
            if (row < p.rows && oc >= 0) idx[e] = prob.out_index(row, oc);
        }
    }
    // FAST with many slices (p.acc): every slice adds its partial into a
    // zeroed accumulator with fire-and-forget L2 reductions; the last
    // arriver reads the sums once, stores C and re-zeroes the accumulator.
    // One L2 round trip instead of nz / FB; the summation order is the
    // arrival order (FAST's contract: within 1e-5 of the reference, not
    // bitwise reproducible).  PARITY never takes this path.
    T* acc = nullptr;
    if constexpr (!PARITY) acc = static_cast<T*>(p.acc);
    if (acc != nullptr) {
        if (owner)
#pragma unroll
            for (int e = 0; e < TILE; ++e)
                if (e < n && idx[e] >= 0) atomicAdd(acc + idx[e], blk[e]);
        __threadfence();
    } else if (owner) {
#pragma unroll
        for (int e = 0; e < TILE; ++e)
            if (e < n && idx[e] >= 0) __stcg(ws + std::int64_t(g) * p.out_elems + idx[e], blk[e]);
    }
    __shared__ int s_last;
    // bar.sync orders every thread's partial stores before thread 0's
    // gpu-scope release (cumulative); its acquire half orders the folding
    // slice's loads after every other slice's stores
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned* ctr = reinterpret_cast<unsigned*>(p.flags) + tile_id;
        unsigned prev;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;\n" : "=r"(prev) : "l"(ctr) : "memory");
        const int last = int(prev) + 1 == p.nz;
        if (last) asm volatile("st.relaxed.gpu.global.u32 [%0], 0;\n" ::"l"(ctr) : "memory");
        s_last = last;
    }
    __syncthreads();
    if (!s_last || !owner) return;
    if (acc != nullptr) {
#pragma unroll
        for (int e = 0; e < TILE; ++e)
            if (e < n && idx[e] >= 0) {
                out[idx[e]] = __ldcg(acc + idx[e]);
                __stcg(acc + idx[e], T(0));
            }
        return;
    }
    // Batches of FB slices: up to 16 independent L2 loads in flight, then the
    // adds in slice order (the order is what parity fixes, not the loads).
    // Wider batches were measured slower: the kernel's register count is set
    // by its peak, and the extra fold registers cost resident blocks.
    T v[TILE];
#pragma unroll
    for (int e = 0; e < TILE; ++e) v[e] = T(0);
    constexpr int FB = TILE >= 16 ? 1 : 16 / TILE;
    for (int g0 = 0; g0 < p.nz; g0 += FB) {
        T part[FB][TILE];
#pragma unroll
        for (int f = 0; f < FB; ++f) {
            const int gg = g0 + f;
            const T* src = ws + std::int64_t(gg) * p.out_elems;
#pragma unroll
            for (int e = 0; e < TILE; ++e)
                part[f][e] = (gg < p.nz && gg != g && e < n && idx[e] >= 0) ? __ldcg(src + idx[e]) : blk[e];
        }
#pragma unroll
        for (int f = 0; f < FB; ++f)
            if (g0 + f < p.nz)
#pragma unroll
                for (int e = 0; e < TILE; ++e)
                    if (e < n) v[e] = A::add(v[e], part[f][e]);
    }
#pragma unroll
    for (int e = 0; e < TILE; ++e)
        if (e < n && idx[e] >= 0) out[idx[e]] = v[e];
}

// Generic (runtime-tile) kernels keep accumulators in local memory up to this
// many per thread; larger register tiles are rejected at launch.
constexpr int kGenericMaxAcc = 256;

template <int MS, int NS, int KS>
struct LaunchCap {
    // Keep the register budget honest: big register tiles only with few threads.
    static constexpr int acc = (MS == 0) ? kGenericMaxAcc : MS * NS * KS;
    static constexpr int threads = (MS == 0) ? 1024 : (acc <= 16 ? 1024 : (acc <= 32 ? 512 : 256));
};

// ARM: the A tile is staged row-major [row][kk] (global A contiguous along
// the reduction, GEMM non-transposed A); otherwise k-major [kk][row].
// BRM: the B tile is staged [col][kk] (GEMM transposed B); otherwise [kk][col].
// Each operand is copied with cp.async chunks of 2^lv elements along its
// global contiguous dimension, so smem keeps that dimension contiguous.
// NARROW instantiations are bounded at 256 threads per block, which lifts the
// register cap from 64 to 255 for small register tiles (software-pipelined
// shared-memory reads, no spills in the k_g fold); the host picks them
// whenever the tuple needs <= 256 threads.
constexpr int kNarrowThreads = 256;

template <class Prob, typename T, int MS_, int NS_, int KS_, bool PARITY, bool ARM, bool BRM, bool NARROW = false>
__global__ void __launch_bounds__(NARROW ? kNarrowThreads : LaunchCap<MS_, NS_, KS_>::threads)
    simt_kernel(const Prob prob, const SimtParams p) {
    constexpr bool RT = (MS_ == 0);  // runtime-tile generic kernel
    const int MS = RT ? p.ms : MS_;
    const int NS = RT ? p.ns : NS_;
    const int KS = RT ? p.ks : KS_;
    constexpr int ACC = RT ? kGenericMaxAcc : (MS_ * NS_ * KS_);
    constexpr int TILE = RT ? kGenericMaxAcc : (MS_ * NS_);
    using A = Arith<T, PARITY>;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    // smem: [col_base nl i64][col_out nl i64][stages x (A all groups, B all groups)]
    std::int64_t* col_base = reinterpret_cast<std::int64_t*>(smem_raw);
    std::int64_t* col_out = col_base + p.nl;
    T* stage_mem = reinterpret_cast<T*>(col_out + p.nl);
    const int stage_elems = p.a_stage + p.b_stage;

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

    simt_probe(p, 0);
    for (int x = tid; x < p.nl; x += nthreads) prob.column(ct, x, col_base[x], col_out[x]);
    __syncthreads();

    // ---- stage loader --------------------------------------------------------
    auto load_a = [&]<int BYTES>(std::int64_t st, T* dst) {
        constexpr int V = BYTES / int(sizeof(T));
        const int lchunks = p.lml + p.lw - p.lva;  // log2 chunks per group
        const int total = p.kl << lchunks;
        const int inner = ARM ? (p.lw - p.lva) : (p.lml - p.lva);
        for (int e = tid; e < total; e += nthreads) {
            const int gx = e >> lchunks;
            const int c = e & ((1 << lchunks) - 1);
            const int outer = c >> inner;
            const int in = (c & ((1 << inner) - 1)) << p.lva;
            const int ii = ARM ? outer : in;
            const int kk = ARM ? in : outer;
            const std::int64_t glo = min(s_hi, s_lo + gx * kl_span);
            const std::int64_t ghi = min(s_hi, glo + kl_span);
            const std::int64_t t = glo + st * p.w + kk;
            const std::int64_t row = row0 + ii;
            int n;
            if constexpr (ARM) n = row < p.rows ? int(max(std::int64_t(0), min(std::int64_t(V), ghi - t))) : 0;
            else n = t < ghi ? int(max(std::int64_t(0), min(std::int64_t(V), p.rows - row))) : 0;
            const T* src = n > 0 ? prob.a_addr(row, t) : reinterpret_cast<const T*>(p.out);
            T* d = dst + gx * p.a_group + (ARM ? ii * p.a_ld + kk : kk * p.a_ld + ii);
            cp_async_zfill<BYTES>(d, src, n * int(sizeof(T)));
        }
    };
    auto load_b = [&]<int BYTES>(std::int64_t st, T* dst) {
        constexpr int V = BYTES / int(sizeof(T));
        const int lchunks = p.lnl + p.lw - p.lvb;
        const int total = p.kl << lchunks;
        const int inner = BRM ? (p.lw - p.lvb) : (p.lnl - p.lvb);
        for (int e = tid; e < total; e += nthreads) {
            const int gx = e >> lchunks;
            const int c = e & ((1 << lchunks) - 1);
            const int outer = c >> inner;
            const int in = (c & ((1 << inner) - 1)) << p.lvb;
            const int xx = BRM ? outer : in;
            const int kk = BRM ? in : outer;
            const std::int64_t glo = min(s_hi, s_lo + gx * kl_span);
            const std::int64_t ghi = min(s_hi, glo + kl_span);
            const std::int64_t t = glo + st * p.w + kk;
            const std::int64_t base = col_base[xx];
            int n;
            if constexpr (BRM) n = base >= 0 ? int(max(std::int64_t(0), min(std::int64_t(V), ghi - t))) : 0;
            else n = t < ghi ? prob.b_cols_valid(base, V) : 0;
            const T* src = n > 0 ? prob.b_addr(t, base) : reinterpret_cast<const T*>(p.out);
            T* d = dst + gx * p.b_group + (BRM ? xx * p.b_ld + kk : kk * p.b_ld + xx);
            cp_async_zfill<BYTES>(d, src, n * int(sizeof(T)));
        }
    };
    // ---- precomputed chunk state (affine problems, host-checked envelope) ----
    ChunkLd ca[kChunkMax], cb[kChunkMax];
    int nca = 0, ncb = 0;
    std::int64_t a_wk = 0, b_wk = 0;  // element advance of one step
    const T* a_origin = prob.a_addr(0, 0);
    if constexpr (Prob::kAffineA) {
        if (p.fast_ld) {
            a_wk = std::int64_t(p.w) * prob.a_kstride();
            {
                const int VA = 1 << p.lva;
                const int lchunks = p.lml + p.lw - p.lva;
                const int total = p.kl << lchunks;
                const int inner = ARM ? (p.lw - p.lva) : (p.lml - p.lva);
                nca = min(kChunkMax, max(0, (total - tid + nthreads - 1) / nthreads));
#pragma unroll
                for (int i = 0; i < kChunkMax; ++i) {
                    if (i >= nca) break;
                    const int e = tid + i * nthreads;
                    const int gx = e >> lchunks;
                    const int c = e & ((1 << lchunks) - 1);
                    const int outer = c >> inner;
                    const int in = (c & ((1 << inner) - 1)) << p.lva;
                    const int ii = ARM ? outer : in;
                    const int kk = ARM ? in : outer;
                    const std::int64_t glo = min(s_hi, s_lo + gx * kl_span);
                    const std::int64_t ghi = min(s_hi, glo + kl_span);
                    const std::int64_t t0 = glo + kk;
                    const std::int64_t row = row0 + ii;
                    const bool rv = row < p.rows;
                    ca[i].off = rv ? int(prob.a_addr(row, t0) - a_origin) : 0;
                    ca[i].dst = gx * p.a_group + (ARM ? ii * p.a_ld + kk : kk * p.a_ld + ii);
                    ca[i].lim = int(ghi - t0);
                    ca[i].cnt = ARM ? (rv ? VA : 0) : int(max(std::int64_t(0), min(std::int64_t(VA), p.rows - row)));
                }
            }
        }
    }
    if constexpr (Prob::kAffine) {
        if (p.fast_ld) {
            b_wk = std::int64_t(p.w) * prob.b_kstride();
            {
                const int VB = 1 << p.lvb;
                const int lchunks = p.lnl + p.lw - p.lvb;
                const int total = p.kl << lchunks;
                const int inner = BRM ? (p.lw - p.lvb) : (p.lnl - p.lvb);
                ncb = min(kChunkMax, max(0, (total - tid + nthreads - 1) / nthreads));
#pragma unroll
                for (int i = 0; i < kChunkMax; ++i) {
                    if (i >= ncb) break;
                    const int e = tid + i * nthreads;
                    const int gx = e >> lchunks;
                    const int c = e & ((1 << lchunks) - 1);
                    const int outer = c >> inner;
                    const int in = (c & ((1 << inner) - 1)) << p.lvb;
                    const int xx = BRM ? outer : in;
                    const int kk = BRM ? in : outer;
                    const std::int64_t glo = min(s_hi, s_lo + gx * kl_span);
                    const std::int64_t ghi = min(s_hi, glo + kl_span);
                    const std::int64_t t0 = glo + kk;
                    const std::int64_t base = col_base[xx];
                    cb[i].off = base >= 0 ? int(prob.b_addr(t0, base) - prob.b) : 0;
                    cb[i].dst = gx * p.b_group + (BRM ? xx * p.b_ld + kk : kk * p.b_ld + xx);
                    cb[i].lim = int(ghi - t0);
                    cb[i].cnt = BRM ? (base >= 0 ? VB : 0) : prob.b_cols_valid(base, VB);
                }
            }
        }
    }
    // ---- precomputed gather state (CONV image operand) ------------------------
    // Per chunk: its column base (or < 0 outside the tensor), first reduction
    // index and the columns left in its group; a step only adds st*w and
    // decomposes the tap (ConvProblem::off).  The reduction index of the
    // gather fits in 32 bits (host-checked).
    struct GatherLd {
        std::int64_t base;
        int t0, lim, dst;
    };
    GatherLd cgs[kChunkMax];
    int ncg = 0;
    bool gather_fast = false;
    if constexpr (!Prob::kAffine) {
        const int lchunks = p.lnl + p.lw - p.lvb;
        const int total = p.kl << lchunks;
        if (p.gather_ld && (total + nthreads - 1) / nthreads <= kChunkMax) {
            gather_fast = true;
            const int inner = BRM ? (p.lw - p.lvb) : (p.lnl - p.lvb);
            ncg = max(0, (total - tid + nthreads - 1) / nthreads);
#pragma unroll
            for (int i = 0; i < kChunkMax; ++i) {
                if (i >= ncg) break;
                const int e = tid + i * nthreads;
                const int gx = e >> lchunks;
                const int c = e & ((1 << lchunks) - 1);
                const int outer = c >> inner;
                const int in = (c & ((1 << inner) - 1)) << p.lvb;
                const int xx = BRM ? outer : in;
                const int kk = BRM ? in : outer;
                const std::int64_t glo = min(s_hi, s_lo + gx * kl_span);
                const std::int64_t ghi = min(s_hi, glo + kl_span);
                cgs[i].base = col_base[xx];
                cgs[i].t0 = int(glo + kk);
                cgs[i].lim = int(ghi - (glo + kk));
                cgs[i].dst = gx * p.b_group + (BRM ? xx * p.b_ld + kk : kk * p.b_ld + xx);
            }
        }
    }
    auto load_gather = [&]<int BYTES>(std::int64_t st, T* dst) {
        if constexpr (!Prob::kAffine) {
            constexpr int V = BYTES / int(sizeof(T));
            const int dk = int(st) * p.w;
            const T* dummy = reinterpret_cast<const T*>(p.out);
#pragma unroll
            for (int i = 0; i < kChunkMax; ++i) {
                if (i < ncg) {
                    const int r = cgs[i].lim - dk;
                    const std::int64_t base = cgs[i].base;
                    int n;
                    if constexpr (BRM) n = base >= 0 ? min(max(r, 0), V) : 0;
                    else n = r > 0 ? prob.b_cols_valid(base, V) : 0;
                    const T* src = n > 0 ? prob.b_addr(cgs[i].t0 + dk, base) : dummy;
                    cp_async_zfill<BYTES>(dst + cgs[i].dst, src, n * int(sizeof(T)));
                }
            }
        }
    };
    auto load_fast_a = [&]<int BA>(std::int64_t st, T* dst) {
        if constexpr (Prob::kAffineA) {
            const int dk = int(st) * p.w;
            const T* dummy = reinterpret_cast<const T*>(p.out);
#pragma unroll
            for (int i = 0; i < kChunkMax; ++i) {
                if (i < nca) {
                    const int r = ca[i].lim - dk;
                    const int n = ARM ? min(max(r, 0), ca[i].cnt) : (r > 0 ? ca[i].cnt : 0);
                    const T* src = n > 0 ? a_origin + (ca[i].off + st * a_wk) : dummy;
                    cp_async_zfill<BA>(dst + ca[i].dst, src, n * int(sizeof(T)));
                }
            }
        }
    };
    auto load_fast = [&]<int BA, int BB>(std::int64_t st, T* dst) {
        if constexpr (Prob::kAffine) {
            const int dk = int(st) * p.w;
            const T* dummy = reinterpret_cast<const T*>(p.out);
            load_fast_a.template operator()<BA>(st, dst);
#pragma unroll
            for (int i = 0; i < kChunkMax; ++i) {
                if (i < ncb) {
                    const int r = cb[i].lim - dk;
                    const int n = BRM ? min(max(r, 0), cb[i].cnt) : (r > 0 ? cb[i].cnt : 0);
                    const T* src = n > 0 ? prob.b + (cb[i].off + st * b_wk) : dummy;
                    cp_async_zfill<BB>(dst + p.a_stage + cb[i].dst, src, n * int(sizeof(T)));
                }
            }
        }
    };
    auto load_stage = [&](std::int64_t st, int slot) {
        T* dst = stage_mem + slot * stage_elems;
        if constexpr (Prob::kAffine) {
            if (p.fast_ld) {
                constexpr int E = int(sizeof(T));
                const int ba = E << p.lva, bb = E << p.lvb;
                if (ba == 16 && bb == 16) load_fast.template operator()<16, 16>(st, dst);
                else if (ba == 16 && bb == E) load_fast.template operator()<16, E>(st, dst);
                else if (ba == E && bb == 16) load_fast.template operator()<E, 16>(st, dst);
                else if (ba == 16 && bb == 8) load_fast.template operator()<16, 8>(st, dst);
                else if (ba == 8 && bb == 16) load_fast.template operator()<8, 16>(st, dst);
                else if (ba == 8 && bb == 8) load_fast.template operator()<8, 8>(st, dst);
                else if (ba == 8 && bb == E) load_fast.template operator()<8, E>(st, dst);
                else if (ba == E && bb == 8) load_fast.template operator()<E, 8>(st, dst);
                else load_fast.template operator()<E, E>(st, dst);
                return;
            }
        }
        if (Prob::kAffineA && p.fast_ld) {
            switch (int(sizeof(T)) << p.lva) {
                case 16: load_fast_a.template operator()<16>(st, dst); break;
                case 8: load_fast_a.template operator()<8>(st, dst); break;
                default: load_fast_a.template operator()<int(sizeof(T))>(st, dst); break;
            }
        } else {
            switch (int(sizeof(T)) << p.lva) {
                case 16: load_a.template operator()<16>(st, dst); break;
                case 8: load_a.template operator()<8>(st, dst); break;
                default: load_a.template operator()<int(sizeof(T))>(st, dst); break;
            }
        }
        if (gather_fast) {
            switch (int(sizeof(T)) << p.lvb) {
                case 16: load_gather.template operator()<16>(st, dst + p.a_stage); break;
                case 8: load_gather.template operator()<8>(st, dst + p.a_stage); break;
                default: load_gather.template operator()<int(sizeof(T))>(st, dst + p.a_stage); break;
            }
            return;
        }
        switch (int(sizeof(T)) << p.lvb) {
            case 16: load_b.template operator()<16>(st, dst + p.a_stage); break;
            case 8: load_b.template operator()<8>(st, dst + p.a_stage); break;
            default: load_b.template operator()<int(sizeof(T))>(st, dst + p.a_stage); break;
        }
    };

    T acc[ACC];
#pragma unroll
    for (int i = 0; i < ACC; ++i) acc[i] = T(0);

    const std::int64_t my_lo = min(s_hi, s_lo + lg * kl_span);
    const std::int64_t my_hi = min(s_hi, my_lo + kl_span);

    // Ownership of rows / columns.  Operands staged contiguous along the
    // reduction (ARM / BRM) are read 16 bytes (VK k-values) at a time per
    // row, so threads own STRIDED rows (distinct rows of a warp fall in
    // distinct bank groups; lanes sharing a row broadcast).  Operands staged
    // contiguous along rows/cols are read as vectors across the thread's own
    // BLOCKED rows/cols.  Ownership never changes what is summed, only who.
    constexpr int VK = 16 / int(sizeof(T));
    auto row_of = [&](int i) { return ARM ? ty + i * p.tm : ty * MS + i; };
    auto col_of = [&](int j) { return BRM ? tx + j * p.tn : tx * NS + j; };

    const int a_ld = p.a_ld, b_ld = p.b_ld;
    const int a_rstep = p.tm * a_ld;  // ARM: distance between a thread's strided rows
    const int b_cstep = p.tn * b_ld;  // BRM: distance between a thread's strided cols

    // ---- multistage cp.async pipeline (one barrier per step) ----------------
    pdl_wait();  // inputs / outputs / workspace may belong to the previous kernel
    const int S = p.stages;
    for (int s = 0; s < S - 1; ++s) {
        if (s < nsteps) load_stage(s, s);
        cp_async_commit();
    }
    // vector path needs VK | w and k_s | VK (set = c % k_s inside a chunk)
    const bool kvec = (KS_ > 0 && KS_ <= VK) && (p.w % VK) == 0;
    int slot = 0;
    simt_probe(p, 1);
    for (std::int64_t st = 0; st < nsteps; ++st) {
        cp_async_wait_dyn(S - 2);
        __syncthreads();
        {
            const std::int64_t nxt = st + S - 1;
            int nslot = slot + S - 1;
            if (nslot >= S) nslot -= S;
            if (nxt < nsteps) load_stage(nxt, nslot);
            cp_async_commit();
        }
        const std::int64_t k0 = my_lo + st * p.w;
        const int nv = int(max(std::int64_t(0), min(std::int64_t(p.w), my_hi - k0)));
        const T* as = stage_mem + slot * stage_elems + lg * p.a_group;
        const T* bs = stage_mem + slot * stage_elems + p.a_stage + lg * p.b_group;
        if constexpr (!RT) {
            if (kvec) {
                // chunks of VK reduction columns; only the tail chunk is
                // predicated (smem past nv holds zero-filled or stale values)
                constexpr int VR = MS_ < VK ? MS_ : VK;  // row vector (k-major A)
                constexpr int VC = NS_ < VK ? NS_ : VK;  // col vector (k-major B)
                using VecK = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
                using Vec2 = typename std::conditional<sizeof(T) == 4, float2, double2>::type;
                const T* a_base = as + (ARM ? ty * a_ld : ty * MS_);
                const T* b_base = bs + (BRM ? tx * b_ld : tx * NS_);
                auto chunk = [&]<bool FULL>(int kk0, int lim) {
                    T ak[ARM ? MS_ * VK : 1];
                    T bk[BRM ? NS_ * VK : 1];
                    if constexpr (ARM) {
#pragma unroll
                        for (int i = 0; i < MS_; ++i) {
                            const VecK v = *reinterpret_cast<const VecK*>(a_base + i * a_rstep + kk0);
                            const T* vp = reinterpret_cast<const T*>(&v);
#pragma unroll
                            for (int c = 0; c < VK; ++c) ak[i * VK + c] = vp[c];
                        }
                    }
                    if constexpr (BRM) {
#pragma unroll
                        for (int j = 0; j < NS_; ++j) {
                            const VecK v = *reinterpret_cast<const VecK*>(b_base + j * b_cstep + kk0);
                            const T* vp = reinterpret_cast<const T*>(&v);
#pragma unroll
                            for (int c = 0; c < VK; ++c) bk[j * VK + c] = vp[c];
                        }
                    }
                    const T* ap = a_base + kk0 * a_ld;
                    const T* bp = b_base + kk0 * b_ld;
#pragma unroll
                    for (int c = 0; c < VK; ++c) {
                        if (FULL || c < lim) {
                            T av[MS_], bv[NS_];
                            if constexpr (ARM) {
#pragma unroll
                                for (int i = 0; i < MS_; ++i) av[i] = ak[i * VK + c];
                            } else {
#pragma unroll
                                for (int i = 0; i < MS_; i += VR) {
                                    if constexpr (VR == 4) {
                                        const float4 v = *reinterpret_cast<const float4*>(ap + i);
                                        av[i] = v.x; av[i + 1] = v.y; av[i + 2] = v.z; av[i + 3] = v.w;
                                    } else if constexpr (VR == 2) {
                                        const Vec2 v = *reinterpret_cast<const Vec2*>(ap + i);
                                        av[i] = v.x; av[i + 1] = v.y;
                                    } else {
                                        av[i] = ap[i];
                                    }
                                }
                            }
                            if constexpr (BRM) {
#pragma unroll
                                for (int j = 0; j < NS_; ++j) bv[j] = bk[j * VK + c];
                            } else {
#pragma unroll
                                for (int j = 0; j < NS_; j += VC) {
                                    if constexpr (VC == 4) {
                                        const float4 v = *reinterpret_cast<const float4*>(bp + j);
                                        bv[j] = v.x; bv[j + 1] = v.y; bv[j + 2] = v.z; bv[j + 3] = v.w;
                                    } else if constexpr (VC == 2) {
                                        const Vec2 v = *reinterpret_cast<const Vec2*>(bp + j);
                                        bv[j] = v.x; bv[j + 1] = v.y;
                                    } else {
                                        bv[j] = bp[j];
                                    }
                                }
                            }
                            constexpr int set_mask = KS_ - 1;  // KS_ divides VK: set = c % KS
#pragma unroll
                            for (int i = 0; i < MS_; ++i)
#pragma unroll
                                for (int j = 0; j < NS_; ++j) {
                                    T& c_ = acc[((c & set_mask) * MS_ + i) * NS_ + j];
                                    c_ = A::mac(c_, av[i], bv[j]);
                                }
                        }
                        if constexpr (!ARM) ap += a_ld;
                        if constexpr (!BRM) bp += b_ld;
                    }
                };
                const int nfull = nv & ~(VK - 1);
                for (int kk0 = 0; kk0 < nfull; kk0 += VK) chunk.template operator()<true>(kk0, VK);
                if (nfull < nv) chunk.template operator()<false>(nfull, nv - nfull);
            } else {
                // narrow stages (w < VK): scalar reads, k_s sets unrolled
                for (int kk0 = 0; kk0 < nv; kk0 += KS_) {
#pragma unroll
                    for (int s = 0; s < KS_; ++s) {
                        const int kk = kk0 + s;
                        if (kk < nv) {
                            T av[MS_], bv[NS_];
#pragma unroll
                            for (int i = 0; i < MS_; ++i)
                                av[i] = ARM ? as[row_of(i) * a_ld + kk] : as[kk * a_ld + row_of(i)];
#pragma unroll
                            for (int j = 0; j < NS_; ++j)
                                bv[j] = BRM ? bs[col_of(j) * b_ld + kk] : bs[kk * b_ld + col_of(j)];
#pragma unroll
                            for (int i = 0; i < MS_; ++i)
#pragma unroll
                                for (int j = 0; j < NS_; ++j) {
                                    T& c_ = acc[(s * MS_ + i) * NS_ + j];
                                    c_ = A::mac(c_, av[i], bv[j]);
                                }
                        }
                    }
                }
            }
        } else {
            // generic runtime-tile kernel: scalar reads, sets iterated at runtime
            for (int kk = 0; kk < nv; ++kk) {
                const int set = kk % KS;  // (k - lo) % k_s since step starts are multiples of w, w % k_s == 0
                for (int i = 0; i < MS; ++i) {
                    const T a_ = ARM ? as[row_of(i) * a_ld + kk] : as[kk * a_ld + row_of(i)];
                    for (int j = 0; j < NS; ++j) {
                        const T b_ = BRM ? bs[col_of(j) * b_ld + kk] : bs[kk * b_ld + col_of(j)];
                        T& c_ = acc[(set * MS + i) * NS + j];
                        c_ = A::mac(c_, a_, b_);
                    }
                }
            }
        }
        if (st == 0) simt_probe(p, 2);
        if (++slot == S) slot = 0;
    }
    cp_async_wait<0>();
    __syncthreads();
    simt_probe(p, 3);
    // main loop done: the next kernel may start its prologue on the SM
    // resources this one no longer needs (earlier, its blocks would compete
    // with this kernel's latency-bound main loop)
    pdl_launch_dependents();

    // ---- fold: k_s sets within a thread, then k_l groups in order ----------
    // (backends.cpp:311-318): blk = ((0 + g0s0) + g0s1) + ... + g1s0 + ...
    T blk[TILE];
    T* red = stage_mem;  // reuse the pipeline smem as an m_l x n_l tile
    const int red_ld = p.nl;
    const bool my_nonempty = my_lo < my_hi;
    for (int step = 0; step < p.kl; ++step) {
        if (lg == step) {
#pragma unroll
            for (int i = 0; i < MS; ++i)
#pragma unroll
                for (int j = 0; j < NS; ++j) {
                    T v = (step == 0) ? T(0) : red[row_of(i) * red_ld + col_of(j)];
                    if (my_nonempty)
#pragma unroll
                        for (int s = 0; s < KS; ++s) v = A::add(v, acc[(s * MS + i) * NS + j]);
                    blk[i * NS + j] = v;
                    if (step + 1 < p.kl) red[row_of(i) * red_ld + col_of(j)] = v;
                }
        }
        __syncthreads();
    }

    simt_probe(p, 4);
    const bool owner = (lg == p.kl - 1);
    simt_store_or_merge<T, PARITY, TILE>(prob, p, blk, MS * NS, owner, [&](int e, std::int64_t& row, std::int64_t& oc) {
        const int i = e / NS, j = e - (e / NS) * NS;
        row = row0 + row_of(i);
        oc = col_out[col_of(j)];
    });
}

}  // namespace ktune_dev
