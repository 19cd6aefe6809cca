// umma.cu -- K4: the tensor-core GEMM family for sm_100a (bf16 / f16 / tf32
// inputs, fp32 accumulation in TMEM, fp32 output).
//
// Replaces execute_gemm (backends.cpp:228-329) for the new dtypes.  Per CTA:
//   warp 0      TMA producer: one elected lane streams A/B tiles into a ring
//               of `stages` shared-memory slots (cp.async.bulk.tensor.2d,
//               128/64/32-byte hardware swizzle, mbarrier complete_tx);
//   warp 1      MMA issuer: allocates TMEM, one elected lane issues
//               tcgen05.mma (kind::f16 or kind::tf32) per UMMA_K slice and
//               frees each slot with tcgen05.commit;
//   warps 2..5  epilogue: tcgen05.ld 32x32b rows of the fp32 accumulator,
//               predicated vector stores (or split-K partial publication).
//
// ISAAC tuple -> tensor-core tile (the legality formulas of param_space.cpp
// stay the space definition; tc_plan() adds the launchability rules):
//   m_l   BLOCK_M: 64 or 128 = UMMA_M of one CTA, 256 = a CTA pair
//         (tcgen05.mma.cta_group::2, 128 rows per CTA)
//   n_l   BLOCK_N = UMMA_N (16..256)
//   u     BLOCK_K elements per pipeline stage (>= 32 bytes)
//   k_g   split-K degree: k_g > 1 runs stream-K over min(SMs, tiles * k_g)
//         CTAs (equal contiguous shares of the (tile, k-block) iterations;
//         split tiles folded by the last-arriving segments, two levels,
//         deterministic order)
//   k_s   TMEM accumulator buffers (1, or 2 = the epilogue of one tile
//         overlaps the MMAs of the next in the persistent schedule)
//   n_s   rasterisation width: concurrent CTAs sweep n_s column tiles
//   k_l   reserved for CTA pairs (must be 1); m_s unused
// Operand majors follow the GEMM layout: A K-major unless trans_a, B
// MN-major unless trans_b (both majors are native tcgen05 descriptor modes
// for 16-bit and tf32 inputs).

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

struct TcParams {
    int M, N, K;
    int bm, bn, bk;
    int tile_m;                   // output rows per tile: 128, or 256 for a CTA pair
    int stages;
    int kb_total;                 // k-blocks per tile
    int streamk;                  // k_g > 1: balanced contiguous (tile, k-block) ranges per CTA
    int csplit;                   // > 1: the k_g slices of a tile are one cluster, reduced through DSMEM
    int deal_rotate;              // deal TMA boxes round-robin across stages (else box b -> warp b % kProducers)
    long long total_it;           // tiles * kb_total (stream-K iteration space)
    int smax, gmax;               // stream-K: max segments per tile, max fold groups per tile
    int a_kmajor, b_kmajor;
    int a_sw, b_sw;               // swizzle span (bytes) of each operand's tiles
    int a_boxes, b_boxes;         // TMA boxes per stage
    int a_rows, b_rows;           // rows per K-major box actually streamed (<= bm / bn per CTA)
    unsigned a_box_bytes, b_box_bytes;
    unsigned a_tile_bytes, b_tile_bytes;  // per stage, 1024-aligned
    unsigned a_box_stride, b_box_stride;  // smem distance between boxes of one stage
    unsigned idesc;
    int umma_k_bytes;             // 32 (UMMA_K elements * element size)
    int esize;
    int tmem_cols;
    int nacc;                     // TMEM accumulator buffers (k_s)
    int tiles_m, tiles_n;         // output tile grid
    int raster;                   // rasterisation group width in n-tiles
    float* C;
    float* ws;                    // [smax][M*N] segment partials (C layout)
    float* ws2;                   // [gmax][M*N] fold-group partials
    unsigned* counters;           // zeroed: [tiles * (pair ? 2 : 1)][gmax + 1] arrival counters
    unsigned a_desc_hi, b_desc_hi;    // SBO | version | layout (descriptor bits 32..63)
    unsigned a_desc_lbo, b_desc_lbo;  // LBO field in place (descriptor bits 16..29)
    unsigned a_koff[8], b_koff[8];    // byte offset of UMMA_K slice kk inside a stage tile
    long long* dbg;  // optional timeline probe (CTA 0): [kb][0]=producer issue, [kb][1]=mma start
};


// warps 0..kProducers-1: TMA producers (a TMA issue occupies its warp for a
// few hundred cycles, so the boxes of a stage are dealt round-robin over
// several warps: measured per-SM ingest scales with the issuing warps);
// warp kProducers: MMA issuer; warps 4..7: epilogue (TMEM lane quarters 0..3)
constexpr int kProducers = 3;
constexpr int kMmaWarp = 3;
constexpr int kEpi0 = 128;  // first epilogue thread
constexpr int kThreads = 256;

// Debug timeline (KTUNE_TC_DEBUG=<device pointer>): %globaltimer of events of
// the CTAs with blockIdx.x = blockIdx.y = 0, 8 slots per grid slice.
__device__ __forceinline__ void probe(const TcParams& p, int slot) {
    if (p.dbg == nullptr || blockIdx.x != 0 || blockIdx.y != 0) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.dbg[blockIdx.z * 8 + slot] = (long long)t;
}

// Work unit u -> (tile, grid slice): slices of one tile are consecutive
// units, so the last slice of a tile always has the largest index (the
// ordered fold may wait on lower units only; with every CTA resident and
// units taken in increasing order per CTA, the waits cannot deadlock).
// Tiles are rasterised in column groups of p.raster n-tiles: the CTAs that
// run concurrently share a few B panels and a few A panels, keeping both in
// L2 instead of re-streaming all of B every wave.
struct Unit {
    int m0, n0, g, tile;
};

__device__ __forceinline__ void probe_kb(const TcParams& p, int i, int slot) {
    if (p.dbg == nullptr || blockIdx.x > 1 || i >= 64) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.dbg[64 + (blockIdx.x * 64 + i) * 4 + slot] = (long long)t;
}

// Output tile t in raster order -> (m0, n0, tile id).
__device__ __forceinline__ Unit unit_of(const TcParams& p, int t) {
    Unit w;
    w.g = 0;
    const int per_group = p.raster * p.tiles_m;
    const int group = t / per_group;
    const int cols = min(p.raster, p.tiles_n - group * p.raster);
    const int local = t - group * per_group;
    const int mt = local / cols;
    const int nt = group * p.raster + local % cols;
    w.m0 = mt * p.tile_m;
    w.n0 = nt * p.bn;
    w.tile = mt * p.tiles_n + nt;
    return w;
}

// ---- stream-K work split (k_g > 1) -------------------------------------------
// The (tile, k-block) iterations of the whole GEMM, tile-major in raster
// order, are cut into G equal contiguous ranges, one per CTA (or pair): every
// SM streams the same number of k-blocks whatever the tile count.  A range
// that covers part of a tile produces a segment; segment j of tile t is the
// one starting in CTA cfind(t*kbt) + j.  Segments of a split tile publish
// partials; the last to arrive in each fold group of kFoldGroup segments
// folds them (segment order), and the last group folds the groups (group
// order) into C: a deterministic two-level fold with no waiting.
constexpr int kFoldGroup = 8;

struct Seg {
    int m0, n0, tile;
    int kb0, kb1;  // k-block range inside the tile
    int j, S;      // segment index within the tile, segments of the tile
};

// last CTA whose range starts at or before iteration i
__device__ __forceinline__ int cfind(long long i, long long T, int G) {
    return int(((i + 1) * G - 1) / T);
}

template <class F>
__device__ __forceinline__ void for_each_seg(const TcParams& p, int cta, int ncta, F&& fn) {
    const int tiles = p.tiles_m * p.tiles_n;
    if (p.csplit > 1) {
        // cluster split: cluster c owns tile c, rank r its r-th contiguous K share
        const int C = p.csplit, t = cta / C, r = cta - t * C;
        if (t < tiles) {
            const Unit w = unit_of(p, t);
            fn(Seg{w.m0, w.n0, w.tile, int((long long)r * p.kb_total / C), int((long long)(r + 1) * p.kb_total / C), r,
                   C});
        }
        return;
    }
    if (!p.streamk) {
        for (int t = cta; t < tiles; t += ncta) {
            const Unit w = unit_of(p, t);
            fn(Seg{w.m0, w.n0, w.tile, 0, p.kb_total, 0, 1});
        }
        return;
    }
    const long long T = p.total_it;
    const int kbt = p.kb_total;
    long long it = (long long)cta * T / ncta;
    const long long e = (long long)(cta + 1) * T / ncta;
    while (it < e) {
        const int t = int(it / kbt);
        const int kb0 = int(it - (long long)t * kbt);
        const int kb1 = int(min((long long)kbt, kb0 + (e - it)));
        const int c0 = cfind((long long)t * kbt, T, ncta);
        const Unit w = unit_of(p, t);
        fn(Seg{w.m0, w.n0, w.tile, kb0, kb1, cta - c0, cfind((long long)(t + 1) * kbt - 1, T, ncta) - c0 + 1});
        it += kb1 - kb0;
    }
}

// PAIR: a cluster of two CTAs on one TPC computes a 256-row tile with
// tcgen05.mma.cta_group::2 issued by the leader (rank 0).  Each CTA stages
// its own 128 rows of A and half of the tile's B columns, so per CTA the
// operand traffic per k-block is (128 + n_l/2) * u instead of (128 + n_l) * u
// -- the L2 -> SM bandwidth (~42 B/clk/SM) is what caps the single-CTA tile.
// Both CTAs' TMA bytes complete on the leader's full barrier; the leader's
// commits arrive on both CTAs' empty / accumulator barriers (multicast), and
// every epilogue thread of the pair arrives on the leader's acc_empty.
template <int KIND, int KSTEPS, bool PAIR>
__global__ void __launch_bounds__(kThreads, 1)
    umma_gemm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                     const TcParams p) {
    if (threadIdx.x == 0) probe(p, 0);
    pdl_launch_dependents();
    if (threadIdx.x == 0 && p.dbg != nullptr) {  // per-CTA start / end (debug timeline)
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.dbg[1024 + blockIdx.x * 4] = (long long)t;
    }
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-align the tile region (SW128 atoms repeat every 1024 bytes).
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                           ~std::uintptr_t(1023));
    const unsigned stage_bytes = p.a_tile_bytes + p.b_tile_bytes;
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + std::size_t(p.stages) * stage_bytes);
    unsigned long long* empty = full + p.stages;
    unsigned long long* acc_full = empty + p.stages;   // [nacc] MMA -> epilogue
    unsigned long long* acc_empty = acc_full + 2;      // [nacc] epilogue -> MMA
    unsigned* tmem_slot = reinterpret_cast<unsigned*>(acc_empty + 2);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const unsigned rank = PAIR ? cluster_ctarank() : 0u;
    const int cta = PAIR ? int(blockIdx.x >> 1) : int(blockIdx.x);   // pair (or CTA) index
    const int ncta = PAIR ? int(gridDim.x >> 1) : int(gridDim.x);
    const bool leader = rank == 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < p.stages; ++s) {
            // one arrive.expect_tx per producer warp (pair: the leader's
            // producers expect both CTAs' bytes of their boxes)
            mbar_init(full + s, kProducers);
            mbar_init(empty + s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(acc_full + a, 1);
            mbar_init(acc_empty + a, PAIR ? 256 : 128);  // every epilogue thread of the CTA (pair)
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<std::uint64_t>(&tma_a)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<std::uint64_t>(&tma_b)) : "memory");
    }
    if (warp == kMmaWarp) {
        if constexpr (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(p.tmem_cols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(p.tmem_cols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    if constexpr (PAIR) cluster_sync();  // peer barriers initialised before anyone signals them
    else __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const unsigned tmem_base = *tmem_slot;
    if (threadIdx.x == 0) probe(p, 1);
    pdl_wait();  // setup above overlaps the previous kernel; global work starts here

    if (warp < kProducers) {
        // ---------------- TMA producers (each warp loops, one lane issues) ----------------
        // Boxes are dealt round-robin over the producer warps across stages
        // (box b of the stage whose first box has running index s goes to
        // warp (s + b) % kProducers): a TMA issue occupies its warp for a few
        // hundred cycles, so with fewer boxes per stage than producers every
        // warp still issues every few stages.  Every producer arrives on each
        // stage's full barrier with the bytes of its own boxes, possibly none
        // (x2 for a pair: the follower issues the same boxes onto the
        // leader's barrier).
        int stage = 0;
        unsigned phase = 0;
        const int a_box_elems = p.a_sw / p.esize, b_box_elems = p.b_sw / p.esize;
        const int nbox = p.a_boxes + p.b_boxes;
        int b_first = warp;  // this warp's first box of the current stage
        const int nbox_mod = p.deal_rotate ? nbox % kProducers : 0;
        const int a_row = PAIR ? int(rank) * 128 : 0;                 // this CTA's rows of the tile
        const int b_col = PAIR ? int(rank) * (p.bn / 2) : 0;          // this CTA's half of the columns
        int dbg_i = 0;
        bool first = true;
        for_each_seg(p, cta, ncta, [&](const Seg& w) {
            for (int kb = w.kb0; kb < w.kb1; ++kb, ++dbg_i) {
                mbar_wait(empty + stage, phase ^ 1u);
                if (lane == 0 && warp == 0) probe_kb(p, dbg_i, 0);
                if (elect_one()) {
                    if (first && warp == 0) probe(p, 2);
                    first = false;
                    unsigned char* sa = smem + std::size_t(stage) * stage_bytes;
                    unsigned char* sb = sa + p.a_tile_bytes;
                    unsigned my_bytes = 0;
                    for (int b = b_first; b < nbox; b += kProducers)
                        my_bytes += b < p.a_boxes ? p.a_box_bytes : p.b_box_bytes;
                    const int k0 = kb * p.bk;
                    const int m0 = w.m0 + a_row, n0 = w.n0 + b_col;
                    if constexpr (PAIR) {
                        const unsigned bar = mapa_shared(smem_u32(full + stage), 0);  // the leader's
                        // the follower's bytes may land before the leader's expect_tx:
                        // the phase cannot complete until the leader's producers arrive
                        if (leader) mbar_expect_tx(full + stage, 2 * my_bytes);
                        for (int b = b_first; b < nbox; b += kProducers) {
                            if (b < p.a_boxes) {
                                const int j = b;
                                if (p.a_kmajor) tma_load_2d_pair(sa + j * p.a_box_stride, &tma_a, bar, k0 + j * a_box_elems, m0);
                                else tma_load_2d_pair(sa + j * p.a_box_stride, &tma_a, bar, m0 + j * a_box_elems, k0);
                            } else {
                                const int j = b - p.a_boxes;
                                if (p.b_kmajor) tma_load_2d_pair(sb + j * p.b_box_stride, &tma_b, bar, k0 + j * b_box_elems, n0);
                                else tma_load_2d_pair(sb + j * p.b_box_stride, &tma_b, bar, n0 + j * b_box_elems, k0);
                            }
                        }
                        if (warp == 0) probe_kb(p, dbg_i, 1);
                    } else {
                        mbar_expect_tx(full + stage, my_bytes);
                        for (int b = b_first; b < nbox; b += kProducers) {
                            if (b < p.a_boxes) {
                                const int j = b;
                                if (p.a_kmajor)
                                    tma_load_2d(sa + j * p.a_box_stride, &tma_a, full + stage, k0 + j * a_box_elems, m0);
                                else
                                    tma_load_2d(sa + j * p.a_box_stride, &tma_a, full + stage, m0 + j * a_box_elems, k0);
                            } else {
                                const int j = b - p.a_boxes;
                                if (p.b_kmajor)
                                    tma_load_2d(sb + j * p.b_box_stride, &tma_b, full + stage, k0 + j * b_box_elems, n0);
                                else
                                    tma_load_2d(sb + j * p.b_box_stride, &tma_b, full + stage, n0 + j * b_box_elems, k0);
                            }
                        }
                    }
                }
                __syncwarp();
                b_first -= nbox_mod;  // the next stage's boxes start nbox later in the deal
                if (b_first < 0) b_first += kProducers;
                if (++stage == p.stages) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        });
    } else if (warp == kMmaWarp) {
        // ---------------- MMA issuer (whole warp loops, one lane issues) ----------------
        // Descriptors: constant high words and k-slice offsets come from the
        // host; per k-block only the 14-bit start address changes.  With
        // nacc = 2 the accumulator alternates between two TMEM column ranges,
        // so the epilogue of one unit overlaps the MMAs of the next.  In a
        // pair only the leader issues (for both CTAs).
        if (leader) {
            int stage = 0;
            unsigned phase = 0;
            int acc = 0;
            unsigned acc_phase = 0;
            int dbg_i = 0;
            const unsigned base = smem_u32(smem);
            bool first = true;
            for_each_seg(p, cta, ncta, [&](const Seg& w) {
                const int nkb = w.kb1 - w.kb0;
                mbar_wait(acc_empty + acc, acc_phase ^ 1u);
                asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                const unsigned d_tmem = tmem_base + unsigned(acc * p.bn);
                for (int i = 0; i < nkb; ++i, ++dbg_i) {
                    mbar_wait(full + stage, phase);
                    if (lane == 0) probe_kb(p, dbg_i, 2);
                    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                    if (elect_one()) {
                        if (i == 0 && first) probe(p, 3);
                        const unsigned sa = base + unsigned(stage) * stage_bytes;
                        const unsigned sb = sa + p.a_tile_bytes;
#pragma unroll
                        for (int kk = 0; kk < KSTEPS; ++kk) {
                            const std::uint64_t adesc = (std::uint64_t(p.a_desc_hi) << 32) |
                                                        (((sa + p.a_koff[kk]) >> 4) & 0x3FFFu) | p.a_desc_lbo;
                            const std::uint64_t bdesc = (std::uint64_t(p.b_desc_hi) << 32) |
                                                        (((sb + p.b_koff[kk]) >> 4) & 0x3FFFu) | p.b_desc_lbo;
                            if constexpr (PAIR) umma_pair<KIND>(d_tmem, adesc, bdesc, p.idesc, (i > 0 || kk > 0) ? 1u : 0u);
                            else umma<KIND>(d_tmem, adesc, bdesc, p.idesc, (i > 0 || kk > 0) ? 1u : 0u);
                        }
                        // slot is free (in both CTAs) once these MMAs retire
                        if constexpr (PAIR) umma_commit_pair(empty + stage);
                        else umma_commit(empty + stage);
                    }
                    __syncwarp();
                    if (++stage == p.stages) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                if (elect_one()) {
                    if (first) probe(p, 4);
                    if constexpr (PAIR) umma_commit_pair(acc_full + acc);
                    else umma_commit(acc_full + acc);
                }
                first = false;
                __syncwarp();
                if (++acc == p.nacc) {
                    acc = 0;
                    acc_phase ^= 1u;
                }
            });
        }
    } else {
        // ---------------- epilogue (warps 4..7) ----------------
        const int quarter = warp & 3;  // TMEM lane quarter this warp may access
        const std::int64_t MN = std::int64_t(p.M) * p.N;
        const int chunk = p.bn >= 32 ? 32 : 16;
        const unsigned acc_empty_leader0 = PAIR ? mapa_shared(smem_u32(acc_empty), 0) : smem_u32(acc_empty);
        const bool vec_ok = ((MN & 3) == 0) && ((reinterpret_cast<std::uintptr_t>(p.C) & 15) == 0) && ((p.N & 3) == 0);
        __shared__ int s_last;
        int acc = 0;
        unsigned acc_phase = 0;
        bool first = true;
        for_each_seg(p, cta, ncta, [&](const Seg& w) {
            // accumulator row -> TMEM lane: M = 128 (and each CTA of a pair):
            // row r in lane r; M = 64: rows 16q..16q+15 in lanes 32q..32q+15
            // of warp quarter q (the upper 16 lanes of each quarter unused)
            const int row = p.bm == 64 ? w.m0 + quarter * 16 + lane : w.m0 + int(rank) * 128 + quarter * 32 + lane;
            const bool row_ok = row < p.M && (p.bm == 64 ? lane < 16 : true);
            const bool csplit = p.csplit > 1;
            const bool split = w.S > 1 && !csplit;
            mbar_wait(acc_full + acc, acc_phase);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            if (threadIdx.x == kEpi0 && first) probe(p, 5);
            if (threadIdx.x == kEpi0 && p.dbg != nullptr) {  // per-CTA: accumulator ready (last segment)
                unsigned long long tt;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
                p.dbg[1024 + blockIdx.x * 4 + 1] = (long long)tt;
            }
            // a split tile's segment goes to its partial slot j, else straight to C
            float* out = split ? p.ws + std::int64_t(w.j) * MN : p.C;
            for (int c0 = 0; c0 < p.bn; c0 += chunk) {
                float v[32];
                const unsigned taddr = tmem_base + (unsigned(quarter * 32) << 16) + unsigned(acc * p.bn + c0);
                if (chunk == 32) tmem_ld32(taddr, v);
                else tmem_ld16(taddr, v);
                if (c0 + chunk >= p.bn) {
                    // accumulator fully read: hand it back to the MMA warp early
                    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
                    if constexpr (PAIR) mbar_arrive_cluster(acc_empty_leader0 + unsigned(acc) * 8u);
                    else mbar_arrive(acc_empty + acc);
                }
                if (csplit) {
                    if (p.bm == 64 && lane >= 16) continue;
                    // this slice's partial row into its own shared memory (the
                    // pipeline ring is idle: every k-block of the slice has been
                    // consumed); an empty slice contributes zeros
                    float* red = reinterpret_cast<float*>(smem) + (row - w.m0) * p.bn + c0;
                    const bool empty_slice = w.kb1 == w.kb0;
#pragma unroll
                    for (int i = 0; i < 32; i += 4)
                        if (i < chunk)
                            *reinterpret_cast<float4*>(red + i) = empty_slice ? make_float4(0.f, 0.f, 0.f, 0.f)
                                                                              : make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                    continue;
                }
                if (!row_ok) continue;
                const std::int64_t base = std::int64_t(row) * p.N + w.n0 + c0;
                const int ncols = min(chunk, p.N - (w.n0 + c0));
                if (ncols <= 0) continue;
                float* dst = out + base;
                if (ncols == chunk && vec_ok) {
#pragma unroll
                    for (int i = 0; i < 32; i += 4)
                        if (i < chunk) {
                            if (split) __stcg(reinterpret_cast<float4*>(dst + i), make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]));
                            else *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                        }
                } else {
                    for (int i = 0; i < ncols; ++i) {
                        if (split) __stcg(dst + i, v[i]);
                        else dst[i] = v[i];
                    }
                }
            }
            if (++acc == p.nacc) {
                acc = 0;
                acc_phase ^= 1u;
            }
            first = false;
            if (!split) return;
            // ---- two-level fold of the tile's segments (no waiting) -------
            const int ngroups = (w.S + kFoldGroup - 1) / kFoldGroup;
            const int q = w.j / kFoldGroup;
            const int g_lo = q * kFoldGroup, g_hi = min(w.S, g_lo + kFoldGroup);
            const std::int64_t ctile = (PAIR ? std::int64_t(w.tile) * 2 + rank : std::int64_t(w.tile)) * (p.gmax + 1);
            unsigned* ctr_group = p.counters + ctile + q;
            unsigned* ctr_tile = p.counters + ctile + p.gmax;
            // fold slots [lo, hi) of `src` (stride MN) in order into `dstbuf` (this thread's row)
            auto fold = [&](const float* src, int lo, int hi, float* dstbuf, bool to_c) {
                if (!row_ok) return;
                for (int c0 = 0; c0 < p.bn; c0 += 16) {
                    const std::int64_t base = std::int64_t(row) * p.N + w.n0 + c0;
                    const int ncols = min(16, p.N - (w.n0 + c0));
                    if (ncols <= 0) break;
                    float accv[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) accv[i] = 0.f;
                    for (int g0 = lo; g0 < hi; g0 += 8) {
                        float part[8][16];
#pragma unroll
                        for (int f = 0; f < 8; ++f) {
                            const float* sp = src + std::int64_t(g0 + f) * MN + base;
                            const bool live = g0 + f < hi;
                            if (ncols == 16 && vec_ok) {
#pragma unroll
                                for (int i = 0; i < 16; i += 4) {
                                    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
                                    if (live) x = __ldcg(reinterpret_cast<const float4*>(sp + i));
                                    part[f][i] = x.x; part[f][i + 1] = x.y; part[f][i + 2] = x.z; part[f][i + 3] = x.w;
                                }
                            } else {
#pragma unroll
                                for (int i = 0; i < 16; ++i) part[f][i] = (live && i < ncols) ? __ldcg(sp + i) : 0.f;
                            }
                        }
#pragma unroll
                        for (int f = 0; f < 8; ++f)
                            if (g0 + f < hi)
#pragma unroll
                                for (int i = 0; i < 16; ++i) accv[i] = __fadd_rn(accv[i], part[f][i]);
                    }
                    float* dp = dstbuf + base;
                    for (int i = 0; i < ncols; ++i) {
                        if (to_c) dp[i] = accv[i];
                        else __stcg(dp + i, accv[i]);
                    }
                }
            };
            // arrival: bar.sync orders the 128 threads' stores before one
            // thread's cumulative gpu-scope release (acq_rel atomic)
            auto arrive_last = [&](unsigned* ctr, int expected) {
                asm volatile("bar.sync 1, 128;\n" ::: "memory");
                if (threadIdx.x == kEpi0) {
                    unsigned prev;
                    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;\n" : "=r"(prev) : "l"(ctr) : "memory");
                    const int last = int(prev) + 1 == expected;
                    if (last) asm volatile("st.relaxed.gpu.global.u32 [%0], 0;\n" ::"l"(ctr) : "memory");
                    s_last = last;
                }
                asm volatile("bar.sync 1, 128;\n" ::: "memory");
                return s_last != 0;
            };
            const bool last_in_group = arrive_last(ctr_group, g_hi - g_lo);
            if (threadIdx.x == kEpi0 && p.dbg != nullptr) {  // per-CTA: ticket taken
                unsigned long long tt;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
                p.dbg[1024 + blockIdx.x * 4 + 2] = (long long)tt;
            }
            if (!last_in_group) return;
            if (ngroups == 1) {
                fold(p.ws, 0, w.S, p.C, true);
                return;
            }
            fold(p.ws, g_lo, g_hi, p.ws2 + std::int64_t(q) * MN, false);
            if (!arrive_last(ctr_tile, ngroups)) return;
            fold(p.ws2, 0, ngroups, p.C, true);
        });
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    if constexpr (PAIR) cluster_sync();  // the peer's MMAs / smem reads are done before either CTA frees
    else if (p.csplit > 1) {
        // cluster split-K: every slice's partial tile sits in its CTA's shared
        // memory; after one cluster barrier every rank reads its share of the
        // tile from all slices through DSMEM, folds it in rank order
        // (((0 + s_0) + s_1) + ...) and writes C
        if (threadIdx.x == kEpi0) probe(p, 6);
        cluster_sync();
        if (threadIdx.x == 0 && p.dbg != nullptr) {  // per-CTA: every slice's partial is in place
            unsigned long long tt;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
            p.dbg[1024 + blockIdx.x * 4 + 2] = (long long)tt;
        }
        // rank r folds quads [r*Q/C, (r+1)*Q/C) of the tile with all its
        // threads; every quad is summed over the slices in rank order
        const int crank = int(cluster_ctarank());
        const int C = p.csplit;
        const int t = int(blockIdx.x) / C;
        if (t < p.tiles_m * p.tiles_n) {
            const Unit w = unit_of(p, t);
            const int qpr = p.bn / 4, Q = p.bm * qpr;
            const int q1 = (crank + 1) * Q / C;
            const unsigned sbase = smem_u32(smem);
            for (int q = crank * Q / C + int(threadIdx.x); q < q1; q += kThreads) {
                const int lrow = q / qpr, c4 = q - lrow * qpr;
                const int row = w.m0 + lrow, col = w.n0 + c4 * 4;
                if (row >= p.M || col >= p.N) continue;
                float4 x[8];
                unsigned ad[8];
#pragma unroll
                for (int r = 0; r < 8; ++r) ad[r] = r < C ? mapa_shared(sbase + unsigned(q) * 16u, unsigned(r)) : 0u;
#pragma unroll
                for (int r = 0; r < 8; ++r)
                    if (r < C)
                        asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                                     : "=f"(x[r].x), "=f"(x[r].y), "=f"(x[r].z), "=f"(x[r].w)
                                     : "r"(ad[r]));
                float4 acc4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int r = 0; r < 8; ++r)
                    if (r < C) {
                        acc4.x = __fadd_rn(acc4.x, x[r].x);
                        acc4.y = __fadd_rn(acc4.y, x[r].y);
                        acc4.z = __fadd_rn(acc4.z, x[r].z);
                        acc4.w = __fadd_rn(acc4.w, x[r].w);
                    }
                float* dst = p.C + std::int64_t(row) * p.N + col;
                if (col + 4 <= p.N && (reinterpret_cast<std::uintptr_t>(dst) & 15) == 0) {
                    *reinterpret_cast<float4*>(dst) = acc4;
                } else {
                    const float vv[4] = {acc4.x, acc4.y, acc4.z, acc4.w};
                    for (int i = 0; i < 4 && col + i < p.N; ++i) dst[i] = vv[i];
                }
            }
        }
        // execution-only barrier: the peers' shared memory stays alive until
        // every rank has read it (the reads completed into registers above);
        // no release, so the C stores need not be acknowledged first
        asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;\n" ::: "memory");
    } else __syncthreads();
    if (threadIdx.x == 0) probe(p, 7);
    if (threadIdx.x == 0 && p.dbg != nullptr) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.dbg[1024 + blockIdx.x * 4 + 3] = (long long)t;
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        if constexpr (PAIR)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(p.tmem_cols));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(p.tmem_cols));
    }
}

}  // namespace tc
}  // namespace ktune_dev

namespace ktune {
namespace umma {

namespace {

using ktune_dev::tc::TcParams;

using namespace detail;

struct TcPlan {
    TcParams p{};
    dim3 grid;
    std::size_t smem{0};
    std::size_t ws_bytes{0};
    // operand staging (any-shape contract of execute_gemm, backends.cpp:228-329):
    // an operand whose leading dimension is not a 16-byte multiple (TMA) is
    // copied into a padded workspace copy; a tf32 operand in MN-major layout
    // is transposed into a K-major copy (tcgen05 kind::tf32 reads K-major)
    bool stage_a{false}, stage_b{false};
    bool tr_a{false}, tr_b{false};           // transpose while staging
    std::int64_t a_ld{0}, b_ld{0};           // leading dimension (elements) the kernel reads
    std::size_t a_stage_off{0}, b_stage_off{0}, stage_bytes{0};
    int kind{0};
    int ksteps{4};
    bool pair{false};  // m_l = 256: cluster of two CTAs, tcgen05.mma.cta_group::2
};


TcPlan tc_plan(const GemmInput& in, const GemmTuning& t) {
    in.validate();
    t.validate();
    if (t.m_l % t.m_s != 0) throw std::invalid_argument("execute: m_l not divisible by m_s");
    if (t.n_l % t.n_s != 0) throw std::invalid_argument("execute: n_l not divisible by n_s");
    if (t.u % t.k_s != 0) throw std::invalid_argument("execute: u not divisible by k_s");
    const int es = dtype_size_bytes(in.dtype);
    TcPlan pl;
    auto& p = pl.p;
    pl.kind = in.dtype == Dtype::tf32 ? 1 : 0;
    if (t.m_l != 64 && t.m_l != 128 && t.m_l != 256)
        throw unsupported_error("tensor-core family: m_l must be 64 or 128 (one CTA) or 256 (CTA pair), got " +
                                std::to_string(t.m_l));
    pl.pair = t.m_l == 256;
    if (pl.pair && (t.n_l < 32 || t.n_l % 32 != 0))
        throw unsupported_error("tensor-core family: a CTA pair splits n_l in halves of >= 16 columns; n_l must be a "
                                "multiple of 32, got " + std::to_string(t.n_l));
    if (t.n_l < 16 || t.n_l > 256)
        throw unsupported_error("tensor-core family: n_l must lie in [16, 256] (UMMA_N), got " + std::to_string(t.n_l));
    if (t.k_l != 1) throw unsupported_error("tensor-core family: k_l must be 1 in this build");
    if (t.k_s > 2) throw unsupported_error("tensor-core family: k_s (TMEM accumulator buffers) must be 1 or 2");
    if (t.u * es < 32) throw unsupported_error("tensor-core family: u * element size must be >= 32 bytes");
    if (in.m > 0x7fffffff || in.n > 0x7fffffff || in.k > 0x7fffffff)
        throw unsupported_error("tensor-core family: dimensions must fit in 32 bits");
    p.M = int(in.m);
    p.N = int(in.n);
    p.K = int(in.k);
    p.bm = t.m_l == 64 ? 64 : 128;  // rows staged per CTA (a pair covers 256); UMMA_M = 64 for m_l = 64
    p.tile_m = pl.pair ? 256 : p.bm;
    p.bn = t.n_l;
    const int bn_cta = pl.pair ? t.n_l / 2 : t.n_l;  // B columns staged per CTA
    p.bk = t.u;
    p.esize = es;
    p.umma_k_bytes = 32;
    p.a_kmajor = in.trans_a ? 0 : 1;
    p.b_kmajor = in.trans_b ? 1 : 0;
    if (in.dtype == Dtype::tf32) {
        // kind::tf32 tiles are K-major here: stage MN-major operands transposed
        pl.tr_a = !p.a_kmajor;
        pl.tr_b = !p.b_kmajor;
        p.a_kmajor = p.b_kmajor = 1;
    }
    // swizzle spans and TMA boxes
    auto span_for = [](int bytes) { return bytes >= 128 ? 128 : (bytes >= 64 ? 64 : 32); };
    if (p.a_kmajor) {
        p.a_sw = span_for(p.bk * es);
        p.a_boxes = p.bk * es / p.a_sw;
        p.a_box_bytes = unsigned(p.a_sw) * p.bm;
    } else {
        p.a_sw = span_for(p.bm * es);
        if (p.bm * es < p.a_sw) throw unsupported_error("tensor-core family: m_l too small for an MN-major A tile");
        p.a_boxes = p.bm * es / p.a_sw;
        p.a_box_bytes = unsigned(p.a_sw) * p.bk;
    }
    if (p.b_kmajor) {
        p.b_sw = span_for(p.bk * es);
        p.b_boxes = p.bk * es / p.b_sw;
        p.b_box_bytes = unsigned(p.b_sw) * bn_cta;
    } else {
        p.b_sw = span_for(bn_cta * es);
        if (bn_cta * es < p.b_sw) throw unsupported_error("tensor-core family: n_l too small for an MN-major B tile");
        p.b_boxes = bn_cta * es / p.b_sw;
        p.b_box_bytes = unsigned(p.b_sw) * p.bk;
    }
    p.a_box_stride = p.a_box_bytes;
    p.b_box_stride = p.b_box_bytes;
    // A single row tile taller than the matrix (M < m_l, e.g. ICA's 32 rows
    // in a 64-row UMMA tile): stream only the rows that exist.  TMA costs a
    // few cycles per box row whatever its width, and rows past M only feed
    // accumulator rows that are never stored (each D row depends on its own
    // A row), so the stale shared memory there is harmless.  Same for the
    // columns of a K-major B narrower than n_l.
    p.a_rows = p.bm;
    p.b_rows = bn_cta;
    if (p.a_kmajor && !pl.pair && in.m < p.bm) {
        p.a_rows = int(std::min<std::int64_t>(p.bm, ceil_div(in.m, 8) * 8));
        p.a_box_bytes = unsigned(p.a_sw) * unsigned(p.a_rows);
    }
    if (p.b_kmajor && !pl.pair && in.n < bn_cta) {
        p.b_rows = int(std::min<std::int64_t>(bn_cta, ceil_div(in.n, 8) * 8));
        p.b_box_bytes = unsigned(p.b_sw) * unsigned(p.b_rows);
    }
    p.a_tile_bytes = unsigned(ceil_div(std::int64_t(p.a_boxes) * p.a_box_stride, 1024) * 1024);
    p.b_tile_bytes = unsigned(ceil_div(std::int64_t(p.b_boxes) * p.b_box_stride, 1024) * 1024);
    // TMA: global strides must be multiples of 16 bytes
    // leading dimensions the kernel reads (after staging): TMA needs 16-byte
    // multiples; other operands are staged into padded (or transposed) copies
    const int align = 16 / es;
    auto padded = [&](std::int64_t x) { return (x + align - 1) / align * align; };
    const std::int64_t a_ld0 = p.a_kmajor ? in.k : in.m, b_ld0 = p.b_kmajor ? in.k : in.n;
    const std::int64_t a_src_ld = in.trans_a ? in.m : in.k, b_src_ld = in.trans_b ? in.k : in.n;
    pl.stage_a = pl.tr_a || (a_src_ld * es) % 16 != 0;
    pl.stage_b = pl.tr_b || (b_src_ld * es) % 16 != 0;
    pl.a_ld = pl.stage_a ? padded(a_ld0) : a_ld0;
    pl.b_ld = pl.stage_b ? padded(b_ld0) : b_ld0;
    p.kb_total = int(ceil_div(in.k, p.bk));
    const std::size_t stage_bytes = std::size_t(p.a_tile_bytes) + p.b_tile_bytes;
    const std::size_t extra = 1024 + 8 * 32 + 64;  // alignment slack + barriers (2*stages + 4) + tmem slot
    const std::size_t optin = std::size_t(smem_optin());
    int stages = int((optin - extra) / stage_bytes);
    stages = std::min(stages, 8);
    if (stages < 2) throw unsupported_error("tensor-core family: tile does not fit two pipeline stages in shared memory");
    p.stages = stages;
    pl.smem = extra + stage_bytes * std::size_t(stages);
    p.nacc = (t.k_s == 2 && 2 * p.bn <= 512) ? 2 : 1;
    p.tmem_cols = std::max(32, pow2_ceil(p.nacc * p.bn));
    p.tiles_m = int(ceil_div(in.m, p.tile_m));
    p.tiles_n = int(ceil_div(in.n, p.bn));
    p.raster = std::max(1, std::min(p.tiles_n, t.n_s));
    // instruction descriptor: F32 accumulate, operand formats, majors, N>>3, M>>4
    const unsigned fmt = in.dtype == Dtype::bf16 ? 1u : (in.dtype == Dtype::f16 ? 0u : 2u);
    p.idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (unsigned(p.a_kmajor ? 0 : 1) << 15) |
              (unsigned(p.b_kmajor ? 0 : 1) << 16) | (unsigned(p.bn >> 3) << 17) |
              (unsigned((pl.pair ? 256 : p.bm) >> 4) << 24);
    // Shared-memory matrix descriptors (tcgen05 "version 1"): high word =
    // SBO (8 rows x swizzle span) | version 1 | swizzle layout; LBO = 16 B for
    // K-major (unused with swizzle), = box stride between MN atoms for
    // MN-major.  Per UMMA_K slice (32 bytes of K) the start address moves
    // 32 B inside a K-major swizzle atom (next box after sw bytes), or
    // UMMA_K rows of sw bytes for MN-major.
    auto hi_word = [](int sw) {
        const unsigned layout = sw == 128 ? 2u : (sw == 64 ? 4u : 6u);
        return ((unsigned(8 * sw) >> 4) & 0x3FFFu) | (1u << 14) | (layout << 29);
    };
    p.a_desc_hi = hi_word(p.a_sw);
    p.b_desc_hi = hi_word(p.b_sw);
    p.a_desc_lbo = ((p.a_kmajor ? 16u : p.a_box_stride) >> 4 & 0x3FFFu) << 16;
    p.b_desc_lbo = ((p.b_kmajor ? 16u : p.b_box_stride) >> 4 & 0x3FFFu) << 16;
    const int ksteps = p.bk * es / p.umma_k_bytes;
    if (ksteps != 1 && ksteps != 2 && ksteps != 4 && ksteps != 8)
        throw unsupported_error("tensor-core family: u * element size must be 32..256 bytes");
    for (int kk = 0; kk < 8; ++kk) {
        const unsigned kb = unsigned(kk * p.umma_k_bytes);
        p.a_koff[kk] = p.a_kmajor ? (kb / p.a_sw) * p.a_box_stride + kb % p.a_sw : (kb / es) * p.a_sw;
        p.b_koff[kk] = p.b_kmajor ? (kb / p.b_sw) * p.b_box_stride + kb % p.b_sw : (kb / es) * p.b_sw;
    }
    pl.ksteps = ksteps;
    // persistent grid: one CTA (or CTA pair) per SM (shared memory holds
    // one CTA).  k_g = 1: whole tiles round-robin.  k_g > 1: stream-K --
    // min(SMs, tiles * k_g) CTAs each take an equal contiguous share of the
    // (tile, k-block) iterations, so every SM streams the same k-blocks
    const std::int64_t tiles = std::int64_t(p.tiles_m) * p.tiles_n;
    if (tiles > 0x7fffffff) throw unsupported_error("too many output tiles for one launch");
    const std::int64_t slots = pl.pair ? num_sms() / 2 : num_sms();
    p.streamk = t.k_g > 1 ? 1 : 0;
    p.csplit = 0;
    p.deal_rotate = std::getenv("KTUNE_TC_STATIC_DEAL") == nullptr ? 1 : 0;
    // cluster split: when k_g <= 8 and at least two slices of every tile fit
    // the SMs at once, each tile is one cluster of C CTAs -- the largest power of two
    // <= min(k_g, 8) whose clusters are all resident together (like
    // stream-K, k_g caps the workers at what the SMs hold) -- and the slices
    // are reduced through distributed shared memory: no global partials,
    // atomics or fold pass.  Otherwise stream-K.  Resident clusters: pairs
    // fill every SM; clusters of 4 strand a few SMs per GPC (132 of 148 CTAs
    // measured); 8 is held to 3/4 of the SMs.  Odd sizes pack GPCs badly
    // (k_g = 8 as 7-CTA clusters ran a second wave: 14.4 us vs 8.4 us).
    // k_g > 8 asks for more workers than a cluster holds: stream-K (ICA
    // 32x32x60000 at k_g = 32: 64 stream-K CTAs 13 us, 16 clustered 27 us).
    {
        const std::int64_t sms = num_sms();
        int C = 0;
        for (int c = 2; c <= 8 && c <= t.k_g && c <= p.kb_total; c *= 2) {
            const std::int64_t cap = c == 2 ? sms : (c == 4 ? sms * 132 / 148 : sms * 3 / 4);
            if (tiles * c <= cap) C = c;
        }
        if (!pl.pair && t.k_g > 1 && t.k_g <= 8 && C >= 2 &&
            std::size_t(p.bm) * p.bn * 4 <= std::size_t(p.stages) * (std::size_t(p.a_tile_bytes) + p.b_tile_bytes) &&
            std::getenv("KTUNE_TC_NO_CSPLIT") == nullptr) {
            p.csplit = C;
            p.streamk = 0;
        }
    }
    p.total_it = tiles * p.kb_total;
    std::int64_t G = p.streamk ? std::min<std::int64_t>({slots, tiles * t.k_g, p.total_it})
                               : std::min<std::int64_t>(slots, tiles);
    if (p.csplit > 1) G = tiles * p.csplit;
    G = std::max<std::int64_t>(G, 1);
    pl.grid = dim3(unsigned(pl.pair ? 2 * G : G), 1, 1);
    p.smax = 1;
    if (p.streamk) {
        auto cfind = [&](std::int64_t i) { return ((i + 1) * G - 1) / p.total_it; };
        for (std::int64_t tl = 0; tl < tiles; ++tl) {
            const std::int64_t S = cfind((tl + 1) * p.kb_total - 1) - cfind(tl * p.kb_total) + 1;
            p.smax = int(std::max<std::int64_t>(p.smax, S));
        }
    }
    p.gmax = (p.smax + ktune_dev::tc::kFoldGroup - 1) / ktune_dev::tc::kFoldGroup;
    if (p.smax > 1) {
        const std::size_t ctr = std::size_t(tiles) * (pl.pair ? 2 : 1) * std::size_t(p.gmax + 1) * sizeof(unsigned);
        if (ctr > dev::kSplitCounterBytes)
            throw unsupported_error("tensor-core family: stream-K over " + std::to_string(tiles) +
                                    " tiles exceeds the split-K counter region");
        pl.ws_bytes = dev::kSplitCounterBytes +
                      std::size_t(p.smax + p.gmax) * std::size_t(in.m) * std::size_t(in.n) * sizeof(float);
    }
    if (pl.stage_a || pl.stage_b) {
        // staged operand copies after the split-K region (256-byte aligned)
        if (pl.ws_bytes == 0) pl.ws_bytes = dev::kSplitCounterBytes;
        auto take = [&](std::size_t bytes) {
            const std::size_t off = (pl.ws_bytes + 255) / 256 * 256;
            pl.ws_bytes = off + bytes;
            return off;
        };
        if (pl.stage_a)
            pl.a_stage_off = take(std::size_t(pl.a_ld) * std::size_t(p.a_kmajor ? in.m : in.k) * std::size_t(es));
        if (pl.stage_b)
            pl.b_stage_off = take(std::size_t(pl.b_ld) * std::size_t(p.b_kmajor ? in.n : in.k) * std::size_t(es));
    }
    return pl;
}


}  // namespace

// Staging copy: dst (rows x cols, leading dimension ld_dst) from src (row
// major rows x cols with ld_src, or transposed: src is cols x rows); 32x32
// tiles through shared memory so both sides stay coalesced.
template <typename E>
__global__ void stage_kernel(const E* __restrict__ src, std::int64_t ld_src, E* __restrict__ dst, std::int64_t ld_dst,
                             std::int64_t rows, std::int64_t cols, int transpose) {
    __shared__ E tile[32][33];
    const std::int64_t r0 = std::int64_t(blockIdx.y) * 32, c0 = std::int64_t(blockIdx.x) * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    for (int i = ty; i < 32; i += 8) {
        // read: transposed source element (c, r) lives at src[c * ld_src + r]
        const std::int64_t r = transpose ? c0 + i : r0 + i, c = transpose ? r0 + tx : c0 + tx;
        const std::int64_t sr = transpose ? r : r, sc = c;
        const bool ok = transpose ? (r < cols && c < rows) : (r < rows && c < cols);
        tile[i][tx] = ok ? src[sr * ld_src + sc] : E(0);
    }
    __syncthreads();
    for (int i = ty; i < 32; i += 8) {
        const std::int64_t r = r0 + i, c = c0 + tx;
        if (r < rows && c < cols) dst[r * ld_dst + c] = transpose ? tile[tx][i] : tile[i][tx];
    }
}

void stage(const void* src, std::int64_t ld_src, void* dst, std::int64_t ld_dst, std::int64_t rows, std::int64_t cols,
           bool transpose, int es, cudaStream_t s) {
    if (!transpose) {
        dev::check(cudaMemcpy2DAsync(dst, std::size_t(ld_dst) * es, src, std::size_t(ld_src) * es,
                                     std::size_t(cols) * es, std::size_t(rows), cudaMemcpyDeviceToDevice, s),
                   "stage copy");
        return;
    }
    const dim3 grid(unsigned((cols + 31) / 32), unsigned((rows + 31) / 32)), block(32, 8);
    if (es == 4)
        stage_kernel<unsigned><<<grid, block, 0, s>>>(static_cast<const unsigned*>(src), ld_src,
                                                      static_cast<unsigned*>(dst), ld_dst, rows, cols, 1);
    else
        stage_kernel<unsigned short><<<grid, block, 0, s>>>(static_cast<const unsigned short*>(src), ld_src,
                                                            static_cast<unsigned short*>(dst), ld_dst, rows, cols, 1);
    dev::check(cudaGetLastError(), "stage transpose launch");
}

std::size_t gemm_workspace_bytes(const GemmInput& in, const GemmTuning& t) { return tc_plan(in, t).ws_bytes; }

dev::LaunchInfo gemm_launch_info(const GemmInput& in, const GemmTuning& t) {
    TcPlan pl = tc_plan(in, t);
    // the family names the K-split schedule the plan chose
    const char* fam = pl.p.csplit == 2   ? "tcgen05-cluster2"
                      : pl.p.csplit == 4 ? "tcgen05-cluster4"
                      : pl.p.csplit == 8 ? "tcgen05-cluster8"
                      : pl.p.streamk     ? (pl.pair ? "tcgen05-pair-streamk" : "tcgen05-streamk")
                                         : (pl.pair ? "tcgen05-pair" : "tcgen05");
    return dev::LaunchInfo{ktune_dev::tc::kThreads, pl.smem, int(pl.grid.x), int(pl.grid.y), int(pl.grid.z), false,
                           fam};
}

void gemm(const GemmInput& in, const GemmTuning& t, const void* a, const void* b, void* c, void* ws,
          std::size_t ws_bytes, cudaStream_t stream) {
    TcPlan pl = tc_plan(in, t);
    auto& p = pl.p;
    if ((reinterpret_cast<std::uintptr_t>(a) | reinterpret_cast<std::uintptr_t>(b)) % 16 != 0)
        throw unsupported_error("tensor-core family: operand pointers must be 16-byte aligned for TMA");
    p.C = static_cast<float*>(c);
    if (const char* d = std::getenv("KTUNE_TC_DEBUG")) p.dbg = reinterpret_cast<long long*>(std::strtoull(d, nullptr, 0));
    if (pl.ws_bytes > 0 && (ws == nullptr || ws_bytes < pl.ws_bytes))
        throw workspace_error("workspace of " + std::to_string(ws_bytes) + " bytes is smaller than the " +
                              std::to_string(pl.ws_bytes) + " bytes this tuning needs");
    const int es0 = p.esize;
    if (pl.stage_a) {
        // A is M x K (ld K) or, transposed, K x M (ld M); the kernel reads the layout p.a_kmajor says
        void* dst = static_cast<unsigned char*>(ws) + pl.a_stage_off;
        if (p.a_kmajor) stage(a, in.trans_a ? in.m : in.k, dst, pl.a_ld, in.m, in.k, pl.tr_a, es0, stream);
        else stage(a, in.m, dst, pl.a_ld, in.k, in.m, false, es0, stream);
        a = dst;
    }
    if (pl.stage_b) {
        // B is K x N (ld N) or, transposed, N x K (ld K)
        void* dst = static_cast<unsigned char*>(ws) + pl.b_stage_off;
        if (p.b_kmajor) stage(b, in.trans_b ? in.k : in.n, dst, pl.b_ld, in.n, in.k, pl.tr_b, es0, stream);
        else stage(b, in.n, dst, pl.b_ld, in.k, in.n, false, es0, stream);
        b = dst;
    }
    if (p.smax > 1) {
        // arrival counters in the zeroed counter region (kernels.hpp), then
        // the segment and fold-group partials
        p.counters = static_cast<unsigned*>(ws);
        p.ws = reinterpret_cast<float*>(static_cast<unsigned char*>(ws) + dev::kSplitCounterBytes);
        p.ws2 = p.ws + std::size_t(p.smax) * std::size_t(in.m) * std::size_t(in.n);
    }
    const int es = p.esize;
    // A: K-major -> [M][K] rows, boxes {a_sw/es along K, bm}; MN-major -> [K][M], boxes {a_sw/es along M, bk}
    CUtensorMap ma = p.a_kmajor ? make_map(a, in.dtype, in.k, in.m, p.a_sw / es, p.a_rows, p.a_sw, pl.a_ld)
                                : make_map(a, in.dtype, in.m, in.k, p.a_sw / es, p.bk, p.a_sw, pl.a_ld);
    CUtensorMap mb = p.b_kmajor ? make_map(b, in.dtype, in.k, in.n, p.b_sw / es, p.b_rows, p.b_sw, pl.b_ld)
                                : make_map(b, in.dtype, in.n, in.k, p.b_sw / es, p.bk, p.b_sw, pl.b_ld);
    using ktune_dev::tc::umma_gemm_kernel;
#define KTUNE_TC_ROW(K, P)                                                                           \
    {reinterpret_cast<const void*>(&umma_gemm_kernel<K, 1, P>), reinterpret_cast<const void*>(&umma_gemm_kernel<K, 2, P>), \
     reinterpret_cast<const void*>(&umma_gemm_kernel<K, 4, P>), reinterpret_cast<const void*>(&umma_gemm_kernel<K, 8, P>)}
    static const void* const kernels[2][2][4] = {{KTUNE_TC_ROW(0, false), KTUNE_TC_ROW(1, false)},
                                                 {KTUNE_TC_ROW(0, true), KTUNE_TC_ROW(1, true)}};
#undef KTUNE_TC_ROW
    const int ki = pl.ksteps == 1 ? 0 : (pl.ksteps == 2 ? 1 : (pl.ksteps == 4 ? 2 : 3));
    const void* kern = kernels[pl.pair ? 1 : 0][pl.kind][ki];
    {
        static std::mutex mu;
        static std::size_t configured[2][2][4] = {};
        std::lock_guard<std::mutex> lock(mu);
        std::size_t& done = configured[pl.pair ? 1 : 0][pl.kind][ki];
        if (done < pl.smem) {
            dev::check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.smem)),
                       "cudaFuncSetAttribute(umma smem)");
            dev::check(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                            cudaSharedmemCarveoutMaxShared),
                       "cudaFuncSetAttribute(carveout)");
            if (pl.pair)
                dev::check(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0),
                           "cudaFuncSetAttribute(cluster)");
            done = pl.smem;
        }
    }
    void* args[] = {&ma, &mb, &p};
    dev::launch(kern, pl.grid, dim3(ktune_dev::tc::kThreads), args, pl.smem, stream,
                pl.pair ? 2 : (p.csplit > 1 ? p.csplit : 1), pl.pair ? "umma pair launch" : "umma launch");
}

}  // namespace umma
}  // namespace ktune
