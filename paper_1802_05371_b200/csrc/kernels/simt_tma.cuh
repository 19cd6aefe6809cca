// simt_tma.cuh -- K1t: the fp32 SIMT GEMM fed by TMA (sm_100a).
//
// Same tuple mapping, same arithmetic and the same fold order as simt_kernel
// (simt.cuh) -- PARITY stays bit-identical to execute_gemm<float>
// (backends.cpp:228-329) -- but the operand staging is moved off the compute
// threads:
//   * one producer warp issues 2-D TMA boxes (cp.async.bulk.tensor) for every
//     k_l group's A and B tile of a stage and arms the stage's "full"
//     mbarrier with the box bytes; no per-thread LDGSTS address math;
//   * compute warps wait on "full", run the register-tile FFMA loop straight
//     from shared memory and release the stage with one arrive per warp on
//     its "empty" mbarrier -- no block-wide barrier per reduction step, so
//     warps drift freely across the pipeline;
//   * operand tiles contiguous along the reduction (A when not transposed, B
//     when transposed) are TMA-swizzled (32/64/128 B) instead of padded: the
//     strided rows a warp reads at one k land in distinct bank groups.
//
// Host side: launch.cu (`tma_eligible`, `launch_gemm_tma`).  The k_g merge is
// the last-arriving-slice fold shared with simt_kernel (simt.cuh).

#pragma once

#include <cuda.h>

#include "simt.cuh"

namespace ktune_dev {

struct TmaGeom {
    int a_box_bytes;   // bytes of one A box (dense)
    int b_box_bytes;
    int a_box_stride;  // bytes between A boxes of a group (1024-aligned when swizzled)
    int b_box_stride;
    int a_nbox, b_nbox;  // boxes per group per stage (k-contiguous tiles split at 128 B)
    int a_wb, b_wb;      // reduction columns per box (k-contiguous tiles); w otherwise
    int a_lwb, b_lwb;    // log2 of a_wb / b_wb
    int a_rb, b_rb;      // swizzle row bytes (a_wb*es / b_wb*es; 16 = no swizzle) for k-contiguous tiles
    int a_grp, b_grp;    // bytes of one group's A / B region in a stage
    int stage_bytes;     // kl * (a_grp + b_grp)
    int compute_threads; // tm*tn*kl
    int producer_warp;   // warp index of the first TMA producer
    int n_producers;     // TMA producer warps (boxes dealt round-robin: a TMA issue occupies its warp)
    unsigned neg_zero;   // 0x80000000 (-0.0f), opaque to ptxas (see mac2)
    int compute_only;    // measurement aid (KTUNE_SIMT_COMPUTE_ONLY): no TMA, no stage waits -- wrong results
};

__device__ __forceinline__ unsigned tma_smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void tma_mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(tma_smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void tma_mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(tma_smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(tma_smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(tma_smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_box_2d(void* dst, const CUtensorMap* map, unsigned long long* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
            tma_smem_u32(dst)),
        "l"(reinterpret_cast<std::uint64_t>(map)), "r"(tma_smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ float4 tma_lds128(unsigned addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}
// owned rows / cols contiguous along the non-reduction dimension
// (tx * NS + j): an even count starts 8-byte aligned, one LDS.64 per pair
__device__ __forceinline__ float2 tma_lds64(unsigned addr) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];\n" : "=f"(v.x), "=f"(v.y) : "r"(addr));
    return v;
}
__device__ __forceinline__ float tma_lds32(unsigned addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(v) : "r"(addr));
    return v;
}
// ---- packed fp32 (FFMA2 / FMUL2 + FADD2, sm_100) -------------------------
// Two accumulators per 64-bit register pair: one instruction issues two
// multiply-adds, halving the FMA issue slots of the register tile.  PARITY
// keeps the separately rounded multiply and add of the reference
// (backends.cpp:299-306): mul.rn.f32x2 then add.rn.f32x2 round each lane
// exactly like __fmul_rn / __fadd_rn.  A scalar operand is broadcast to both
// lanes ({a, a}), which ptxas encodes as the .F32 operand form (no move).
__device__ __forceinline__ unsigned long long pk2(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float2 up2(unsigned long long v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
// PARITY: the product as fma(a, b, nz) with nz = {-0.0, -0.0} -- exactly
// round(a*b) for every input (x + -0 == x; -0 keeps the sign of a zero
// product) -- then add.rn.f32x2.  ptxas contracts a mul.rn.f32x2 /
// add.rn.f32x2 pair (and an fma with a literal -0) into one FFMA2, which
// would round once; nz arrives from a kernel parameter, so it cannot.
template <bool PARITY>
__device__ __forceinline__ void mac2(unsigned long long& d, unsigned long long a, unsigned long long b,
                                     unsigned long long nz) {
    if constexpr (PARITY) {
        unsigned long long t;
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(t) : "l"(a), "l"(b), "l"(nz));
        asm("add.rn.f32x2 %0, %0, %1;" : "+l"(d) : "l"(t));
    } else {
        asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
    }
}

__device__ __forceinline__ void tma_prefetch_map(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<std::uint64_t>(map)) : "memory");
}

// Byte offset of the 16-byte chunk at (row, chunk c) of a k-contiguous box
// with rb-byte rows after the TMA swizzle (rb in {16, 32, 64, 128}; 16 = no
// swizzle): the chunk index is XORed with bits [7, 7+log2(rb/16)) of the
// dense offset (PTX tensor-copy swizzle modes).
__device__ __forceinline__ int swz_row_xor(int row, int rb) { return ((row * rb) >> 3) & (rb - 16); }

template <typename T, int MS_, int NS_, int KS_, bool PARITY, bool ARM, bool BRM, bool NARROW>
__global__ void __launch_bounds__(NARROW ? kNarrowThreads + 4 * 32 : 1024)
    simt_tma_kernel(const __grid_constant__ CUtensorMap a_map, const __grid_constant__ CUtensorMap b_map,
                    const GemmProblem<T> prob, const SimtParams p, const TmaGeom g) {
    static_assert(MS_ > 0, "register-tile instantiations only");
    static_assert(sizeof(T) == 4, "the TMA feed is compiled for fp32");
    using A = Arith<T, PARITY>;
    constexpr int ES = int(sizeof(T));
    constexpr int VK = 16 / ES;
    constexpr int TILE = MS_ * NS_;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    // [pad to 1024][stages x stage_bytes | fold tile][full[S], empty[S] mbarriers][col_out nl i64]
    // (swizzled boxes need 1024-byte aligned shared addresses; static shared
    // variables may precede the dynamic segment, so align at run time)
    unsigned char* stages_mem = smem_raw + ((1024u - (tma_smem_u32(smem_raw) & 1023u)) & 1023u);
    // barriers + column table after the pipeline or the k_l fold tile, whichever is larger
    const std::size_t tail_off = (max(std::size_t(p.stages) * g.stage_bytes, std::size_t(p.ml) * p.nl * ES) + 15) & ~std::size_t(15);
    unsigned long long* full = reinterpret_cast<unsigned long long*>(stages_mem + tail_off);
    unsigned long long* empty = full + p.stages;
    std::int64_t* col_out = reinterpret_cast<std::int64_t*>(empty + p.stages);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int ct = blockIdx.x, rt = blockIdx.y, gz = blockIdx.z;
    const std::int64_t row0 = std::int64_t(rt) * p.ml;
    const int col0 = ct * p.nl;

    // the reduction fits in 31 bits on this path (host-checked): 32-bit ranges
    const int red_len = int(p.red), kg_span = int(p.kg_span);
    const int s_lo = min(red_len, gz * kg_span);
    const int s_hi = min(red_len, s_lo + kg_span);
    const int kl_span = (s_hi - s_lo + p.kl - 1) / p.kl;
    const int nsteps = (kl_span + p.w - 1) / p.w;
    const int compute_warps = (g.compute_threads + 31) >> 5;

    if (tid == 0) {
        for (int s = 0; s < p.stages; ++s) {
            tma_mbar_init(&full[s], unsigned(g.n_producers));
            tma_mbar_init(&empty[s], unsigned(compute_warps));
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == g.producer_warp && lane == 0) {
        tma_prefetch_map(&a_map);
        tma_prefetch_map(&b_map);
    }
    for (int x = tid; x < p.nl; x += blockDim.x) {
        std::int64_t base, oc;
        prob.column(ct, x, base, oc);
        col_out[x] = oc;
    }
    simt_probe(p, 0);
    __syncthreads();
    pdl_wait();  // operands / output / workspace may belong to the previous kernel
    simt_probe(p, 1);

    // accumulators: packed pairs along the register tile's columns (NS even),
    // else along its rows (MS even), else scalar
    constexpr int PAIR = (NS_ % 2 == 0) ? 1 : ((MS_ % 2 == 0) ? 2 : 0);
    constexpr int NACC = MS_ * NS_ * KS_;
    unsigned long long accp[PAIR ? NACC / 2 : 1];
    T acc[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = T(0);
#pragma unroll
    for (int i = 0; i < (PAIR ? NACC / 2 : 1); ++i) accp[i] = 0ull;

    const int per_group = p.tm * p.tn;
    const int lg = tid / per_group;
    const int r_in = tid - lg * per_group;
    const int ty = r_in / p.tn;
    const int tx = r_in - ty * p.tn;
    auto row_of = [&](int i) { return ARM ? ty + i * p.tm : ty * MS_ + i; };
    auto col_of = [&](int j) { return BRM ? tx + j * p.tn : tx * NS_ + j; };
    const int my_lo = min(s_hi, s_lo + lg * kl_span);
    const int my_hi = min(s_hi, my_lo + kl_span);

    if (warp >= g.producer_warp && !g.compute_only) {
        // ---- TMA producers (one lane each) ------------------------------
        // The boxes of a step -- per live group: A boxes then B boxes -- are
        // dealt round-robin over the producer warps; each arrives on the
        // stage's full barrier with the bytes of its own boxes.
        const int pw = warp - g.producer_warp;
        if (lane == 0) {
            int slot = 0;
            unsigned phase = 0;  // parity of the ring pass (stage reuse count & 1)
            const int per_group = g.a_nbox + g.b_nbox;
            // groups still streaming at step st: those with len(gx) > st*w;
            // lengths are non-increasing in gx (only the last groups run short)
            for (int st = 0; st < nsteps; ++st) {
                if (st >= p.stages) tma_mbar_wait(&empty[slot], phase ^ 1u);
                const int off = st * p.w;
                int live = 0;
                for (int gx = 0; gx < p.kl; ++gx) {
                    const int glo = min(s_hi, s_lo + gx * kl_span);
                    const int ghi = min(s_hi, glo + kl_span);
                    live += (glo + off < ghi) ? 1 : 0;
                }
                unsigned mine = 0;
                for (int b = pw; b < live * per_group; b += g.n_producers)
                    mine += unsigned(b % per_group < g.a_nbox ? g.a_box_bytes : g.b_box_bytes);
                tma_mbar_expect_tx(&full[slot], mine);
                unsigned char* stage = stages_mem + slot * g.stage_bytes;
                for (int b = pw; b < live * per_group; b += g.n_producers) {
                    const int gx = b / per_group, j = b - gx * per_group;
                    const int kc = min(s_hi, s_lo + gx * kl_span) + off;
                    unsigned char* ga = stage + gx * (g.a_grp + g.b_grp);
                    unsigned char* gb = ga + g.a_grp;
                    if (j < g.a_nbox) {
                        if constexpr (ARM) tma_box_2d(ga + j * g.a_box_stride, &a_map, &full[slot], int(kc) + j * g.a_wb, int(row0));
                        else tma_box_2d(ga, &a_map, &full[slot], int(row0), int(kc));
                    } else {
                        const int jb = j - g.a_nbox;
                        if constexpr (BRM) tma_box_2d(gb + jb * g.b_box_stride, &b_map, &full[slot], int(kc) + jb * g.b_wb, col0);
                        else tma_box_2d(gb, &b_map, &full[slot], col0, int(kc));
                    }
                }
                if (++slot == p.stages) {
                    slot = 0;
                    phase ^= 1u;
                }
            }
        }
    } else if (warp < g.producer_warp) {
        // ---- compute warps (lanes past compute_threads only keep the warp
        // whole for __syncwarp and the per-warp stage release) ------------
        // per-thread shared-memory byte offsets of the owned rows / cols
        // (32-bit shared addresses throughout: LDS, no generic addressing)
        const unsigned sbase = tma_smem_u32(stages_mem);
        unsigned a_off[MS_], a_xor[MS_], b_off[NS_], b_xor[NS_];
#pragma unroll
        for (int i = 0; i < MS_; ++i) {
            const int r = row_of(i);
            a_off[i] = unsigned(ARM ? r * g.a_rb : r * ES);
            a_xor[i] = unsigned(ARM ? swz_row_xor(r, g.a_rb) : 0);
        }
#pragma unroll
        for (int j = 0; j < NS_; ++j) {
            const int c = col_of(j);
            b_off[j] = unsigned(BRM ? c * g.b_rb : c * ES);
            b_xor[j] = unsigned(BRM ? swz_row_xor(c, g.b_rb) : 0);
        }
        const unsigned a_kbytes = unsigned(p.ml * ES);  // !ARM: bytes of one reduction row of the A box
        const unsigned b_kbytes = unsigned(p.nl * ES);
        const int a_wmask = g.a_wb - 1, b_wmask = g.b_wb - 1;
        const unsigned long long nz2 = (static_cast<unsigned long long>(g.neg_zero) << 32) | g.neg_zero;
        int slot = 0;
        unsigned phase = 0;
        const int my_len = tid < g.compute_threads ? my_hi - my_lo : 0;
        for (int st = 0; st < nsteps; ++st) {
            const int nv = max(0, min(p.w, my_len - st * p.w));
            if (!g.compute_only) tma_mbar_wait(&full[slot], phase);
            if (st == 0) simt_probe(p, 2);
            const unsigned ga = sbase + unsigned(slot * g.stage_bytes + lg * (g.a_grp + g.b_grp));
            const unsigned gb = ga + unsigned(g.a_grp);
            // WB > 0: box width known at compile time (full steps; a k-contiguous
            // box row holds min(w, 128 / ES) columns), so chunk offsets and box
            // indices fold into constants; WB == 0: runtime widths
            auto chunk = [&]<bool FULL, int WB>(int kk0, int lim) {
                T ak[ARM ? MS_ * VK : 1];
                T bk[BRM ? NS_ * VK : 1];
                if constexpr (ARM) {
                    const unsigned base = WB ? ga + unsigned(kk0 / (WB ? WB : 1)) * unsigned(g.a_box_stride)
                                             : ga + unsigned((kk0 >> g.a_lwb) * g.a_box_stride);
                    const unsigned cb = unsigned((WB ? kk0 % (WB ? WB : 1) : (kk0 & a_wmask)) * ES);
#pragma unroll
                    for (int i = 0; i < MS_; ++i) {
                        const float4 v = tma_lds128(base + a_off[i] + (cb ^ a_xor[i]));
                        ak[i * VK + 0] = v.x; ak[i * VK + 1] = v.y; ak[i * VK + 2] = v.z; ak[i * VK + 3] = v.w;
                    }
                }
                if constexpr (BRM) {
                    const unsigned base = WB ? gb + unsigned(kk0 / (WB ? WB : 1)) * unsigned(g.b_box_stride)
                                             : gb + unsigned((kk0 >> g.b_lwb) * g.b_box_stride);
                    const unsigned cb = unsigned((WB ? kk0 % (WB ? WB : 1) : (kk0 & b_wmask)) * ES);
#pragma unroll
                    for (int j = 0; j < NS_; ++j) {
                        const float4 v = tma_lds128(base + b_off[j] + (cb ^ b_xor[j]));
                        bk[j * VK + 0] = v.x; bk[j * VK + 1] = v.y; bk[j * VK + 2] = v.z; bk[j * VK + 3] = v.w;
                    }
                }
                const unsigned ap0 = ga + unsigned(kk0) * a_kbytes + a_off[0];
                const unsigned bp0 = gb + unsigned(kk0) * b_kbytes + b_off[0];
#pragma unroll
                for (int c = 0; c < VK; ++c) {
                    if (FULL || c < lim) {
                        T av[MS_], bv[NS_];
                        if constexpr (ARM) {
#pragma unroll
                            for (int i = 0; i < MS_; ++i) av[i] = ak[i * VK + c];
                        } else {
                            const unsigned ap = ap0 + unsigned(c) * a_kbytes;
                            if constexpr (MS_ * ES % 16 == 0) {
#pragma unroll
                                for (int i = 0; i < MS_; i += VK) {
                                    const float4 v = tma_lds128(ap + unsigned(i * ES));
                                    av[i] = v.x; av[i + 1] = v.y; av[i + 2] = v.z; av[i + 3] = v.w;
                                }
                            } else if constexpr (MS_ * ES % 8 == 0) {
#pragma unroll
                                for (int i = 0; i < MS_; i += 2) {
                                    const float2 v = tma_lds64(ap + unsigned(i * ES));
                                    av[i] = v.x; av[i + 1] = v.y;
                                }
                            } else {
#pragma unroll
                                for (int i = 0; i < MS_; ++i) av[i] = tma_lds32(ap + unsigned(i * ES));
                            }
                        }
                        if constexpr (BRM) {
#pragma unroll
                            for (int j = 0; j < NS_; ++j) bv[j] = bk[j * VK + c];
                        } else {
                            const unsigned bp = bp0 + unsigned(c) * b_kbytes;
                            if constexpr (NS_ * ES % 16 == 0) {
#pragma unroll
                                for (int j = 0; j < NS_; j += VK) {
                                    const float4 v = tma_lds128(bp + unsigned(j * ES));
                                    bv[j] = v.x; bv[j + 1] = v.y; bv[j + 2] = v.z; bv[j + 3] = v.w;
                                }
                            } else if constexpr (NS_ * ES % 8 == 0) {
#pragma unroll
                                for (int j = 0; j < NS_; j += 2) {
                                    const float2 v = tma_lds64(bp + unsigned(j * ES));
                                    bv[j] = v.x; bv[j + 1] = v.y;
                                }
                            } else {
#pragma unroll
                                for (int j = 0; j < NS_; ++j) bv[j] = tma_lds32(bp + unsigned(j * ES));
                            }
                        }
                        constexpr int set_mask = KS_ - 1;  // KS_ divides VK: set = c % KS
                        const int set = c & set_mask;
                        if constexpr (PAIR == 1) {
#pragma unroll
                            for (int j = 0; j < NS_; j += 2) {
                                const unsigned long long b2 = pk2(bv[j], bv[j + 1]);
#pragma unroll
                                for (int i = 0; i < MS_; ++i)
                                    mac2<PARITY>(accp[((set * MS_ + i) * NS_ + j) / 2], pk2(av[i], av[i]), b2, nz2);
                            }
                        } else if constexpr (PAIR == 2) {
#pragma unroll
                            for (int i = 0; i < MS_; i += 2) {
                                const unsigned long long a2 = pk2(av[i], av[i + 1]);
#pragma unroll
                                for (int j = 0; j < NS_; ++j)
                                    mac2<PARITY>(accp[((set * NS_ + j) * MS_ + i) / 2], a2, pk2(bv[j], bv[j]), nz2);
                            }
                        } else {
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
            };
            // full steps of the common widths run fully unrolled (compile-time
            // smem offsets, loads scheduled ahead of the FFMAs); partial steps
            // and other widths take the runtime loop with a predicated tail
            auto full_step = [&]<int W>() {
                constexpr int WB = W * ES <= 128 ? W : 128 / ES;
#pragma unroll
                for (int kk0 = 0; kk0 < W; kk0 += VK) chunk.template operator()<true, WB>(kk0, VK);
            };
            if (nv == p.w && p.w == 16) full_step.template operator()<16>();
            else if (nv == p.w && p.w == 32) full_step.template operator()<32>();
            else if (nv == p.w && p.w == 8) full_step.template operator()<8>();
            else if (nv == p.w && p.w == 64) full_step.template operator()<64>();
            else {
                const int nfull = nv & ~(VK - 1);
                for (int kk0 = 0; kk0 < nfull; kk0 += VK) chunk.template operator()<true, 0>(kk0, VK);
                if (nfull < nv) chunk.template operator()<false, 0>(nfull, nv - nfull);
            }
            __syncwarp();
            if (lane == 0 && !g.compute_only) tma_mbar_arrive(&empty[slot]);
            if (++slot == p.stages) {
                slot = 0;
                phase ^= 1u;
            }
        }
    }
    // every stage consumed (compute warps waited on each "full"), so all TMA
    // writes have landed: the pipeline memory is reused for the k_l fold
    __syncthreads();
    simt_probe(p, 3);
    pdl_launch_dependents();

    if constexpr (PAIR == 1) {
#pragma unroll
        for (int q = 0; q < NACC / 2; ++q) {
            const float2 v = up2(accp[q]);
            acc[2 * q] = v.x;
            acc[2 * q + 1] = v.y;
        }
    } else if constexpr (PAIR == 2) {  // pairs ordered [set][j][i / 2]
#pragma unroll
        for (int st = 0; st < KS_; ++st)
#pragma unroll
            for (int j = 0; j < NS_; ++j)
#pragma unroll
                for (int i = 0; i < MS_; i += 2) {
                    const float2 v = up2(accp[((st * NS_ + j) * MS_ + i) / 2]);
                    acc[(st * MS_ + i) * NS_ + j] = v.x;
                    acc[(st * MS_ + i + 1) * NS_ + j] = v.y;
                }
    }
    // ---- fold: k_s sets within a thread, then k_l groups in order ----------
    T blk[TILE];
    T* red = reinterpret_cast<T*>(stages_mem);
    const bool compute = tid < g.compute_threads;
    const bool my_nonempty = my_lo < my_hi;
    for (int step = 0; step < p.kl; ++step) {
        if (compute && lg == step) {
#pragma unroll
            for (int i = 0; i < MS_; ++i)
#pragma unroll
                for (int j = 0; j < NS_; ++j) {
                    T v = (step == 0) ? T(0) : red[row_of(i) * p.nl + col_of(j)];
                    if (my_nonempty)
#pragma unroll
                        for (int s = 0; s < KS_; ++s) v = A::add(v, acc[(s * MS_ + i) * NS_ + j]);
                    blk[i * NS_ + j] = v;
                    if (step + 1 < p.kl) red[row_of(i) * p.nl + col_of(j)] = v;
                }
        }
        __syncthreads();
    }
    simt_probe(p, 4);
    const bool owner = compute && (lg == p.kl - 1);
    simt_store_or_merge<T, PARITY, TILE>(prob, p, blk, TILE, owner, [&](int e, std::int64_t& row, std::int64_t& oc) {
        const int i = e / NS_, j = e - (e / NS_) * NS_;
        row = row0 + row_of(i);
        oc = col_out[col_of(j)];
    });
    simt_probe(p, 5);
}

}  // namespace ktune_dev
