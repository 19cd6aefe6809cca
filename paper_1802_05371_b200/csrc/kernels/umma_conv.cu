// umma_conv.cu -- K4c: implicit-GEMM convolution on the tcgen05 tensor cores
// (bf16 / f16 inputs, fp32 accumulation in TMEM, fp32 output).
//
// Replaces execute_conv (backends.cpp:331-432) for the 16-bit dtypes.  The
// reference's CONV is the GEMM  O[k][pqn] = sum_t F[t][k] * I[t][pqn]  over
// t = (c, r, s) with layouts I = C,H,W,N  F = C,R,S,K  O = K,P,Q,N
// (backends.cpp:345-353, the indirection table of :357-368).  On the tensor
// cores the output PIXELS are the MMA's M dimension and the FILTERS its N:
//   D[pixel][filter] (TMEM, lane = pixel) += I[t][pixel]^T * F[t][filter]
// so one accumulator row is one output pixel and the epilogue's stores of a
// filter column are 32 consecutive pixels -> coalesced along O's innermost
// (q, n) run.
//
// Both operands arrive by TMA, which keeps far more bytes in flight per SM
// than a cp.async gather (measured: a 128-thread LDGSTS gather issued one
// 16 KB stage per ~1.5 us L2 round trip, 3x slower than cuDNN).  The trick
// is the reduction ORDER: blocks of u input channels at a fixed filter tap
// (r, s), taps outermost --  t = (r, s, c)  instead of the reference's
// (c, r, s).  For a fixed tap and channel block the 128 pixels of a tile are
// two boxes of I viewed as [C][H][W*N]: rows = channels, each row one
// 128-byte run of the flattened (w, n) axis -- 64 pixels of one output row
// p, shifted by the tap (r, s).  (A TMA box row is padded to the swizzle
// span, so the run must be the whole 128 bytes: n_l == N, or n_l >= 64.)  The
// matching filter rows are a 3-D box of F viewed as [C][RS][K].  TMA zero
// fills channels >= C and image columns past W, so ragged C, Q and N need no
// special casing (pixels past Q/P are computed and dropped by the epilogue).
// The tensor-core family is a fast family -- its summation order is not the
// reference's and it is checked against the double direct convolution.
//
// Per CTA (persistent, one per SM):
//   warp 0      TMA producer: per stage two 64-pixel image boxes (one per
//               128-byte swizzle atom of the MN-major A tile) and the filter
//               boxes, one mbarrier complete_tx;
//   warp 1      MMA issuer (tcgen05.mma kind::f16, one elected lane);
//   warps 2..5  epilogue (tcgen05.ld, coalesced stores along the pixel run,
//               ordered split-K fold).
//
// ISAAC conv tuple -> tile (legality formulas unchanged, conv_plan() adds the
// launchability rules):
//   p_l*q_l*n_l   BLOCK_M = UMMA_M = 128 output pixels; n_l == N (whole
//                 batch) with q_l*n_l >= 64, or n_l >= 64
//   k_l           BLOCK_N = UMMA_N filters (16..256, multiple of 16)
//   u             channels per pipeline stage (16, 32, 64 or 128)
//   c_g           split-K slices over the (tap, channel-block) sequence
//   c_s           TMEM accumulator buffers (1 or 2)
//   c_l           must be 1;  k_s, p_s, q_s, n_s unused (register tiles of
//                 the SIMT family -- the tensor core owns the whole tile)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <string>

#include "umma.hpp"
#include "umma_common.cuh"

namespace ktune_dev {
namespace tc {

struct ConvTcParams {
    int Nb, P, Q, K, C, R, S, H, W;
    int CRS, RS;
    int pl, ql, nl;
    int tiles_p, tiles_q, tiles_nb, tiles_sp, tiles_k;
    int bn, bk, stages;
    int kb_total, kb_span, nz;
    int cblocks;                  // channel blocks of u per filter tap
    int a_org_n[2], a_org_q[2], a_org_p[2];  // box origin of each 64-pixel atom inside the tile
    unsigned a_box_bytes;
    int b_sw, b_boxes;
    unsigned b_box_bytes, b_box_stride;
    unsigned a_tile_bytes, b_tile_bytes, a_box_stride;
    unsigned idesc;
    unsigned a_desc_hi, b_desc_hi, a_desc_lbo, b_desc_lbo;
    unsigned a_koff[8], b_koff[8];
    int tmem_cols, nacc;
    long long PQN;
    float* out;
    float* ws;
    unsigned long long* flags;
    unsigned long long token;
    long long* dbg;  // optional timeline (KTUNE_TC_DEBUG): CTA 0, [i][slot]
};

__device__ __forceinline__ void conv_probe(const ConvTcParams& p, int i, int slot) {
    if (p.dbg == nullptr || blockIdx.x != 0 || i >= 64) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.dbg[i * 4 + slot] = (long long)t;
}

// warps 0..2: TMA producers (a TMA issue occupies its warp for a few hundred
// cycles; the boxes of a stage are dealt round-robin), warp 3: MMA issuer,
// warps 4..7: epilogue (TMEM lane quarters 0..3)
constexpr int kConvProducers = 3;
constexpr int kConvMmaWarp = 3;
constexpr int kConvEpi0 = 128;
constexpr int kConvThreads = 256;

struct ConvUnit {
    int p0, q0, n0, k0, g, tile;
};

// Unit u -> (spatial tile, filter tile, slice).  Slices of one tile are
// consecutive (the ordered fold only waits on lower units); the filter tiles
// of one spatial tile are adjacent so they share the gathered image rows in L2.
__device__ __forceinline__ ConvUnit conv_unit_of(const ConvTcParams& p, int u) {
    ConvUnit w;
    w.g = u % p.nz;
    const int t = u / p.nz;
    const int kt = t % p.tiles_k;
    const int sp = t / p.tiles_k;
    const int nt = sp % p.tiles_nb;
    const int qt = (sp / p.tiles_nb) % p.tiles_q;
    const int pt = sp / (p.tiles_nb * p.tiles_q);
    w.p0 = pt * p.pl;
    w.q0 = qt * p.ql;
    w.n0 = nt * p.nl;
    w.k0 = kt * p.bn;
    w.tile = t;
    return w;
}

template <int KSTEPS>
__global__ void __launch_bounds__(kConvThreads, 1)
    umma_conv_kernel(const __grid_constant__ CUtensorMap tma_i, const __grid_constant__ CUtensorMap tma_f,
                     const ConvTcParams p) {
    pdl_launch_dependents();
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                           ~std::uintptr_t(1023));
    const unsigned stage_bytes = p.a_tile_bytes + p.b_tile_bytes;
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + std::size_t(p.stages) * stage_bytes);
    unsigned long long* empty = full + p.stages;
    unsigned long long* acc_full = empty + p.stages;
    unsigned long long* acc_empty = acc_full + 2;
    unsigned* tmem_slot = reinterpret_cast<unsigned*>(acc_empty + 2);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const int n_units = p.tiles_sp * p.tiles_k * p.nz;

    if (threadIdx.x == 0) {
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(full + s, kConvProducers);  // one arrive.expect_tx per producer warp
            mbar_init(empty + s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(acc_full + a, 1);
            mbar_init(acc_empty + a, 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<std::uint64_t>(&tma_i)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<std::uint64_t>(&tma_f)) : "memory");
    }
    if (warp == kConvMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "r"(p.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const unsigned tmem_base = *tmem_slot;
    pdl_wait();  // setup above overlaps the previous kernel; global work starts here

    if (warp < kConvProducers) {
        // ---------------- TMA producers ----------------
        // Each producer warp walks every k-block of every unit; the boxes (two
        // image atoms, then the filter boxes) are dealt round-robin over the
        // producer warps across stages, as in the GEMM (umma.cu), so every
        // warp issues even when a stage has fewer boxes than producers.  The
        // (tap, channel block) position advances incrementally and the box
        // origins are computed once per unit.
        int stage = 0;
        unsigned phase = 0;
        const int box_elems = p.b_sw / 2;
        const int nbox = 2 + p.b_boxes;
        int b_first = warp;
        const int nbox_mod = nbox % kConvProducers;
        const int Nb = p.Nb, S = p.S, bk = p.bk, cblocks = p.cblocks, b_boxes = p.b_boxes;
        const unsigned a_tile = p.a_tile_bytes, a_box_stride = p.a_box_stride, b_box_stride = p.b_box_stride;
        int dbg_i = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            const ConvUnit w = conv_unit_of(p, u);
            const int kb_begin = w.g * p.kb_span;
            const int kb_end = min(p.kb_total, kb_begin + p.kb_span);
            // image box origins (w*n coordinate before the tap shift, h row)
            const int ax0 = (w.q0 + p.a_org_q[0]) * Nb + w.n0 + p.a_org_n[0];
            const int ax1 = (w.q0 + p.a_org_q[1]) * Nb + w.n0 + p.a_org_n[1];
            const int ah0 = w.p0 + p.a_org_p[0], ah1 = w.p0 + p.a_org_p[1];
            int rs = kb_begin / cblocks;
            int cb = kb_begin - rs * cblocks;
            int r = rs / S, sx = rs - r * S;
            for (int kb = kb_begin; kb < kb_end; ++kb, ++dbg_i) {
                mbar_wait(empty + stage, phase ^ 1u);
                if (lane == 0 && warp == 0) conv_probe(p, dbg_i, 0);
                if (elect_one()) {
                    const int c0 = cb * bk;
                    unsigned char* sa = smem + std::size_t(stage) * stage_bytes;
                    unsigned char* sb = sa + a_tile;
                    unsigned tx_bytes = 0;
                    for (int b = b_first; b < nbox; b += kConvProducers)
                        tx_bytes += b < 2 ? p.a_box_bytes : p.b_box_bytes;
                    mbar_expect_tx(full + stage, tx_bytes);
                    for (int b = b_first; b < 2 + b_boxes; b += kConvProducers) {
                        if (b == 0) tma_load_3d(sa, &tma_i, full + stage, ax0 + sx * Nb, ah0 + r, c0);
                        else if (b == 1) tma_load_3d(sa + a_box_stride, &tma_i, full + stage, ax1 + sx * Nb, ah1 + r, c0);
                        else
                            tma_load_3d(sb + (b - 2) * b_box_stride, &tma_f, full + stage, w.k0 + (b - 2) * box_elems,
                                        rs, c0);
                    }
                    if (warp == 0) conv_probe(p, dbg_i, 2);
                }
                __syncwarp();
                b_first -= nbox_mod;
                if (b_first < 0) b_first += kConvProducers;
                if (++cb == cblocks) {
                    cb = 0;
                    ++rs;
                    if (++sx == S) {
                        sx = 0;
                        ++r;
                    }
                }
                if (++stage == p.stages) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
    } else if (warp == kConvMmaWarp) {
        // ---------------- MMA issuer ----------------
        int stage = 0;
        unsigned phase = 0;
        int acc = 0;
        unsigned acc_phase = 0;
        const unsigned base = smem_u32(smem);
        int dbg_i = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            const ConvUnit w = conv_unit_of(p, u);
            const int kb_begin = w.g * p.kb_span;
            const int nkb = min(p.kb_total, kb_begin + p.kb_span) - kb_begin;
            mbar_wait(acc_empty + acc, acc_phase ^ 1u);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            const unsigned d_tmem = tmem_base + unsigned(acc * p.bn);
            for (int i = 0; i < nkb; ++i, ++dbg_i) {
                mbar_wait(full + stage, phase);
                if (lane == 0) conv_probe(p, dbg_i, 1);
                asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                if (elect_one()) {
                    const unsigned sa = base + unsigned(stage) * stage_bytes;
                    const unsigned sb = sa + p.a_tile_bytes;
#pragma unroll
                    for (int kk = 0; kk < KSTEPS; ++kk) {
                        const std::uint64_t adesc = (std::uint64_t(p.a_desc_hi) << 32) |
                                                    (((sa + p.a_koff[kk]) >> 4) & 0x3FFFu) | p.a_desc_lbo;
                        const std::uint64_t bdesc = (std::uint64_t(p.b_desc_hi) << 32) |
                                                    (((sb + p.b_koff[kk]) >> 4) & 0x3FFFu) | p.b_desc_lbo;
                        umma<0>(d_tmem, adesc, bdesc, p.idesc, (i > 0 || kk > 0) ? 1u : 0u);
                    }
                    umma_commit(empty + stage);
                }
                __syncwarp();
                if (++stage == p.stages) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
            if (elect_one()) umma_commit(acc_full + acc);
            __syncwarp();
            if (++acc == p.nacc) {
                acc = 0;
                acc_phase ^= 1u;
            }
        }
    } else {
        // ---------------- epilogue (warps 2..5) ----------------
        const int quarter = warp & 3;
        const int m = quarter * 32 + lane;  // pixel of the tile this thread stores
        const int nn = m % p.nl;
        const int qq = (m / p.nl) % p.ql;
        const int pp = m / (p.nl * p.ql);
        const long long total = (long long)p.K * p.PQN;
        const std::int64_t tiles = std::int64_t(p.tiles_sp) * p.tiles_k;
        const int chunk = p.bn >= 32 ? 32 : 16;
        int acc = 0;
        unsigned acc_phase = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            const ConvUnit w = conv_unit_of(p, u);
            const bool last = (w.g == p.nz - 1);
            const bool pix_ok = (w.p0 + pp < p.P) && (w.q0 + qq < p.Q) && (w.n0 + nn < p.Nb);
            const long long pix = ((long long)(w.p0 + pp) * p.Q + (w.q0 + qq)) * p.Nb + (w.n0 + nn);
            mbar_wait(acc_full + acc, acc_phase);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            if (threadIdx.x == kConvEpi0) conv_probe(p, 60 + (u / gridDim.x) % 4, 3);
            if (last && p.nz > 1) {
                for (int gg = threadIdx.x - kConvEpi0; gg < p.nz - 1; gg += 128) {
                    unsigned long long* flag = p.flags + std::int64_t(gg) * tiles + w.tile;
                    unsigned long long v;
                    while (true) {
                        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(flag) : "memory");
                        if (v == p.token) {
                            // consumed: clear it, so a re-launch with the same token
                            // (a replayed CUDA graph) waits for its own publication
                            asm volatile("st.relaxed.gpu.global.u64 [%0], %1;\n" ::"l"(flag), "l"(0ull) : "memory");
                            break;
                        }
                        __nanosleep(32);
                    }
                }
                asm volatile("bar.sync 1, 128;\n" ::: "memory");
            }
            for (int c0 = 0; c0 < p.bn; c0 += chunk) {
                float v[32];
                const unsigned taddr = tmem_base + (unsigned(quarter * 32) << 16) + unsigned(acc * p.bn + c0);
                if (chunk == 32) tmem_ld32(taddr, v);
                else tmem_ld16(taddr, v);
                if (c0 + chunk >= p.bn) {
                    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
                    mbar_arrive(acc_empty + acc);
                }
                if (!pix_ok) continue;
                const int ncols = min(chunk, p.K - (w.k0 + c0));
                if (ncols <= 0) continue;
                const long long base = (long long)(w.k0 + c0) * p.PQN + pix;
                if (p.nz == 1 || last) {
                    if (p.nz > 1) {
                        float accv[32];
#pragma unroll
                        for (int i = 0; i < 32; ++i) accv[i] = 0.f;
                        // two slices per batch of in-flight loads, added in slice order
                        constexpr int FB = 2;
                        for (int g0 = 0; g0 < p.nz - 1; g0 += FB) {
                            float part[FB][32];
#pragma unroll
                            for (int f = 0; f < FB; ++f) {
                                const bool live = g0 + f < p.nz - 1;
                                const float* src = p.ws + (g0 + f) * total + base;
#pragma unroll
                                for (int i = 0; i < 32; ++i)
                                    part[f][i] = (live && i < ncols) ? __ldcg(src + i * p.PQN) : 0.f;
                            }
#pragma unroll
                            for (int f = 0; f < FB; ++f)
                                if (g0 + f < p.nz - 1)
#pragma unroll
                                    for (int i = 0; i < 32; ++i) accv[i] = __fadd_rn(accv[i], part[f][i]);
                        }
#pragma unroll
                        for (int i = 0; i < 32; ++i) v[i] = __fadd_rn(accv[i], v[i]);
                    }
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (i < ncols) p.out[base + i * p.PQN] = v[i];
                } else {
                    float* dst = p.ws + std::int64_t(w.g) * total + base;
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (i < ncols) __stcg(dst + i * p.PQN, v[i]);
                }
            }
            if (!last && p.nz > 1) {
                // bar.sync orders the 128 threads' partial stores before one
                // thread's cumulative gpu-scope release (no per-thread fence)
                asm volatile("bar.sync 1, 128;\n" ::: "memory");
                if (threadIdx.x == kConvEpi0) {
                    unsigned long long* flag = p.flags + std::int64_t(w.g) * tiles + w.tile;
                    asm volatile("fence.acq_rel.gpu;\nst.release.gpu.global.u64 [%0], %1;\n" ::"l"(flag), "l"(p.token)
                                 : "memory");
                }
            }
            if (++acc == p.nacc) {
                acc = 0;
                acc_phase ^= 1u;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == kConvMmaWarp) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(p.tmem_cols));
    }
}

}  // namespace tc
}  // namespace ktune_dev

namespace ktune {
namespace umma {

namespace {

using ktune_dev::tc::ConvTcParams;
using namespace detail;

struct ConvPlan {
    ConvTcParams p{};
    dim3 grid;
    std::size_t smem{0};
    std::size_t ws_bytes{0}, flag_bytes{0};
    // filter counts that are not multiples of 8 (TMA needs 16-byte row
    // pitches): the filters are staged into a copy with a padded pitch
    std::int64_t k_ld{0};
    std::size_t f_stage_off{0};
    int ksteps{4};
    int box[3]{};  // image TMA box {w*n, h, c}
};

ConvPlan conv_plan(const ConvInput& in, const ConvTuning& t) {
    in.validate();
    t.validate();
    if (t.k_l % t.k_s != 0) throw std::invalid_argument("execute: k_l not divisible by k_s");
    if (t.p_l % t.p_s != 0) throw std::invalid_argument("execute: p_l not divisible by p_s");
    if (t.q_l % t.q_s != 0) throw std::invalid_argument("execute: q_l not divisible by q_s");
    if (t.n_l % t.n_s != 0) throw std::invalid_argument("execute: n_l not divisible by n_s");
    if (t.u % t.c_s != 0) throw std::invalid_argument("execute: u not divisible by c_s");
    if (in.dtype != Dtype::bf16 && in.dtype != Dtype::f16)
        throw unsupported_error(std::string("tensor-core conv family executes bf16 / f16, not ") + to_string(in.dtype));
    const int es = 2;
    if (std::int64_t(t.p_l) * t.q_l * t.n_l != 128)
        throw unsupported_error("tensor-core conv family: p_l * q_l * n_l must be 128 output pixels (UMMA_M)");
    if (in.n_batch % 8 != 0)
        throw unsupported_error("tensor-core conv family: the batch must be a multiple of 8 (16-byte TMA strides)");
    if (!(t.n_l >= 64 || (t.n_l == in.n_batch && t.q_l * t.n_l >= 64)))
        throw unsupported_error("tensor-core conv family: a 64-pixel atom must be one contiguous (w, n) run: "
                                "n_l == N with q_l * n_l >= 64, or n_l >= 64");
    if (in.w() * in.n_batch > 0x7fffffff)
        throw unsupported_error("tensor-core conv family: W * N must fit in 32 bits");
    if (t.k_l < 16 || t.k_l > 256 || t.k_l % 16 != 0)
        throw unsupported_error("tensor-core conv family: k_l must be a multiple of 16 in [16, 256] (UMMA_N)");
    if (t.c_l != 1) throw unsupported_error("tensor-core conv family: c_l must be 1");
    if (t.c_s > 2) throw unsupported_error("tensor-core conv family: c_s (TMEM accumulator buffers) must be 1 or 2");
    if (t.u != 16 && t.u != 32 && t.u != 64 && t.u != 128)
        throw unsupported_error("tensor-core conv family: u must be 16, 32, 64 or 128");
    const std::int64_t crs = in.c * in.r * in.s;
    const std::int64_t pqn = in.p * in.q * in.n_batch;
    if (crs > 0x7fffffff || in.k_filters > 0x7fffffff || in.h() * in.w() > 0x7fffffff ||
        in.k_filters * pqn > (std::int64_t(1) << 46))
        throw unsupported_error("tensor-core conv family: problem too large for one launch");
    ConvPlan pl;
    auto& p = pl.p;
    pl.box[0] = 64;
    pl.box[1] = 1;
    pl.box[2] = t.u;
    p.Nb = int(in.n_batch);
    p.P = int(in.p);
    p.Q = int(in.q);
    p.K = int(in.k_filters);
    p.C = int(in.c);
    p.R = int(in.r);
    p.S = int(in.s);
    p.H = int(in.h());
    p.W = int(in.w());
    p.CRS = int(crs);
    p.RS = int(in.r * in.s);
    p.pl = t.p_l;
    p.ql = t.q_l;
    p.nl = t.n_l;
    p.tiles_p = int(ceil_div(in.p, t.p_l));
    p.tiles_q = int(ceil_div(in.q, t.q_l));
    p.tiles_nb = int(ceil_div(in.n_batch, t.n_l));
    const std::int64_t tiles_sp = std::int64_t(p.tiles_p) * p.tiles_q * p.tiles_nb;
    p.tiles_k = int(ceil_div(in.k_filters, t.k_l));
    p.bn = t.k_l;
    p.bk = t.u;
    p.PQN = pqn;
    // A (image): 128 pixels x u channels as two 64-pixel SW128 atoms; each
    // atom is one TMA box {64, 1, u} of I viewed as [C][H][W*N] -> one
    // 128-byte row (64 pixels in tile order) per channel
    for (int j = 0; j < 2; ++j) {
        const int m0 = 64 * j;
        p.a_org_n[j] = m0 % t.n_l;
        p.a_org_q[j] = (m0 / t.n_l) % t.q_l;
        p.a_org_p[j] = m0 / (t.n_l * t.q_l);
    }
    p.a_box_bytes = unsigned(p.bk) * 128u;
    p.a_box_stride = p.a_box_bytes;
    p.a_tile_bytes = unsigned(ceil_div(2 * std::int64_t(p.a_box_stride), 1024) * 1024);
    // B (filters, TMA): MN-major boxes of b_sw bytes x u rows
    p.b_sw = p.bn * es >= 128 ? 128 : (p.bn * es >= 64 ? 64 : 32);
    p.b_boxes = p.bn * es / p.b_sw;
    p.b_box_bytes = unsigned(p.b_sw) * p.bk;
    p.b_box_stride = p.b_box_bytes;
    p.b_tile_bytes = unsigned(ceil_div(std::int64_t(p.b_boxes) * p.b_box_bytes, 1024) * 1024);
    p.cblocks = int(ceil_div(in.c, p.bk));
    p.kb_total = int(in.r * in.s) * p.cblocks;  // (tap, channel block), taps outermost
    p.kb_span = int(ceil_div(p.kb_total, t.c_g));
    p.nz = int(ceil_div(p.kb_total, p.kb_span));
    const std::size_t stage_bytes = std::size_t(p.a_tile_bytes) + p.b_tile_bytes;
    const std::size_t extra = 1024 + 8 * 32 + 64;
    int stages = int((std::size_t(smem_optin()) - extra) / stage_bytes);
    stages = std::min(stages, 8);
    if (stages < 2)
        throw unsupported_error("tensor-core conv family: tile does not fit enough pipeline stages in shared memory");
    p.stages = stages;
    pl.smem = extra + stage_bytes * std::size_t(stages);
    p.nacc = (t.c_s == 2 && 2 * p.bn <= 512) ? 2 : 1;
    p.tmem_cols = std::max(32, pow2_ceil(p.nacc * p.bn));
    const unsigned fmt = in.dtype == Dtype::bf16 ? 1u : 0u;
    // both operands MN-major (pixels resp. filters contiguous), M = 128
    p.idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (1u << 15) | (1u << 16) | (unsigned(p.bn >> 3) << 17) |
              (unsigned(128 >> 4) << 24);
    auto hi_word = [](int sw) {
        const unsigned layout = sw == 128 ? 2u : (sw == 64 ? 4u : 6u);
        return ((unsigned(8 * sw) >> 4) & 0x3FFFu) | (1u << 14) | (layout << 29);
    };
    p.a_desc_hi = hi_word(128);
    p.b_desc_hi = hi_word(p.b_sw);
    p.a_desc_lbo = ((p.a_box_stride >> 4) & 0x3FFFu) << 16;
    p.b_desc_lbo = ((p.b_box_stride >> 4) & 0x3FFFu) << 16;
    pl.ksteps = p.bk / 16;  // UMMA_K = 16 elements = 32 bytes
    for (int kk = 0; kk < 8; ++kk) {
        p.a_koff[kk] = unsigned(kk * 16) * 128u;
        p.b_koff[kk] = unsigned(kk * 16) * unsigned(p.b_sw);
    }
    const std::int64_t units = tiles_sp * p.tiles_k * p.nz;
    if (units > 0x7fffffff) throw unsupported_error("too many work units for one launch");
    p.tiles_sp = int(tiles_sp);
    pl.grid = dim3(unsigned(std::min<std::int64_t>(units, num_sms())), 1, 1);
    if (p.nz > 1) {
        pl.flag_bytes = (std::size_t(tiles_sp) * p.tiles_k * std::size_t(p.nz - 1) * 8 + 255) / 256 * 256;
        pl.ws_bytes = dev::kSplitCounterBytes + pl.flag_bytes + std::size_t(p.nz - 1) * std::size_t(in.k_filters) * std::size_t(pqn) * 4;
    }
    pl.k_ld = (in.k_filters + 7) / 8 * 8;
    if (pl.k_ld != in.k_filters) {
        if (pl.ws_bytes == 0) pl.ws_bytes = dev::kSplitCounterBytes;
        pl.f_stage_off = (pl.ws_bytes + 255) / 256 * 256;
        pl.ws_bytes = pl.f_stage_off + std::size_t(crs) * std::size_t(pl.k_ld) * es;
    }
    return pl;
}

}  // namespace

std::size_t conv_workspace_bytes(const ConvInput& in, const ConvTuning& t) { return conv_plan(in, t).ws_bytes; }

dev::LaunchInfo conv_launch_info(const ConvInput& in, const ConvTuning& t) {
    ConvPlan pl = conv_plan(in, t);
    return dev::LaunchInfo{ktune_dev::tc::kConvThreads, pl.smem, int(pl.grid.x), int(pl.grid.y), int(pl.grid.z),
                           false, "tcgen05-conv"};
}

void conv(const ConvInput& in, const ConvTuning& t, const void* images, const void* filters, void* outputs, void* ws,
          std::size_t ws_bytes, cudaStream_t stream) {
    ConvPlan pl = conv_plan(in, t);
    auto& p = pl.p;
    if ((reinterpret_cast<std::uintptr_t>(images) | reinterpret_cast<std::uintptr_t>(filters)) % 16 != 0)
        throw unsupported_error("tensor-core conv family: image and filter pointers must be 16-byte aligned");
    if (const char* d = std::getenv("KTUNE_TC_DEBUG")) p.dbg = reinterpret_cast<long long*>(std::strtoull(d, nullptr, 0));
    p.out = static_cast<float*>(outputs);
    if (pl.ws_bytes > 0 && (ws == nullptr || ws_bytes < pl.ws_bytes))
        throw workspace_error("workspace of " + std::to_string(ws_bytes) + " bytes is smaller than the " +
                              std::to_string(pl.ws_bytes) + " bytes this tuning needs");
    if (pl.k_ld != in.k_filters) {
        void* dst = static_cast<unsigned char*>(ws) + pl.f_stage_off;
        dev::check(cudaMemcpy2DAsync(dst, std::size_t(pl.k_ld) * 2, filters, std::size_t(in.k_filters) * 2,
                                     std::size_t(in.k_filters) * 2, std::size_t(in.c * in.r * in.s),
                                     cudaMemcpyDeviceToDevice, stream),
                   "stage filters");
        filters = dst;
    }
    if (p.nz > 1) {
        // past the SIMT family's zeroed counter region (kernels.hpp)
        p.flags = reinterpret_cast<unsigned long long*>(static_cast<unsigned char*>(ws) + dev::kSplitCounterBytes);
        p.ws = reinterpret_cast<float*>(static_cast<unsigned char*>(ws) + dev::kSplitCounterBytes + pl.flag_bytes);
        p.token = next_token();
    }
    // images I[c][h][w][n] -> 3-D map {W*N, H, C}; filters F[c][rs][k] -> 3-D map {K, RS, C}
    const std::int64_t idims[3] = {in.w() * in.n_batch, in.h(), in.c};
    CUtensorMap mi = make_map_nd(images, in.dtype, 3, idims, pl.box, 128);
    const std::int64_t fdims[3] = {in.k_filters, in.r * in.s, in.c};
    const int fbox[3] = {p.b_sw / 2, 1, p.bk};
    CUtensorMap mf = make_map_nd(filters, in.dtype, 3, fdims, fbox, p.b_sw, pl.k_ld);
    using ktune_dev::tc::umma_conv_kernel;
    static const void* const kernels[4] = {
        reinterpret_cast<const void*>(&umma_conv_kernel<1>), reinterpret_cast<const void*>(&umma_conv_kernel<2>),
        reinterpret_cast<const void*>(&umma_conv_kernel<4>), reinterpret_cast<const void*>(&umma_conv_kernel<8>)};
    const int ki = pl.ksteps == 1 ? 0 : (pl.ksteps == 2 ? 1 : (pl.ksteps == 4 ? 2 : 3));
    const void* kern = kernels[ki];
    {
        static std::mutex mu;
        static std::size_t configured[4] = {};
        std::lock_guard<std::mutex> lock(mu);
        if (configured[ki] < pl.smem) {
            dev::check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.smem)),
                       "cudaFuncSetAttribute(umma conv smem)");
            dev::check(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                            cudaSharedmemCarveoutMaxShared),
                       "cudaFuncSetAttribute(carveout)");
            dev::check(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                            cudaSharedmemCarveoutMaxShared),
                       "cudaFuncSetAttribute(carveout)");
            configured[ki] = pl.smem;
        }
    }
    void* args[] = {&mi, &mf, &p};
    dev::launch(kern, pl.grid, dim3(ktune_dev::tc::kConvThreads), args, pl.smem, stream, 1, "umma conv launch");
}

}  // namespace umma
}  // namespace ktune
