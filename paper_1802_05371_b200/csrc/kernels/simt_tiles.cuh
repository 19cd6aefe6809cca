// simt_tiles.cuh -- the register-tile envelope compiled ahead of time.
//
// GEMM (MS=m_s, NS=n_s, KS=k_s): MS,NS in {1,2,4,8}, KS in {1,2,4},
//   MS*NS*KS <= 128.  CONV (MS=k_s, NS=p_s*q_s*n_s, KS=c_s): MS in {1,2,4,8},
//   NS in {1,2,4,8,16}, KS in {1,2}, product <= 128.  Everything outside runs
//   on the runtime-tile generic instantiation (MS=NS=KS=0).
#pragma once

#define KTUNE_GEMM_TILES_KS(X, KS) \
    X(1, 1, KS) X(1, 2, KS) X(2, 1, KS) X(1, 4, KS) X(2, 2, KS) X(4, 1, KS) X(1, 8, KS) X(2, 4, KS) X(4, 2, KS) \
    X(8, 1, KS) X(2, 8, KS) X(4, 4, KS) X(8, 2, KS) X(4, 8, KS) X(8, 4, KS)

#define KTUNE_GEMM_TILES(X) \
    KTUNE_GEMM_TILES_KS(X, 1) KTUNE_GEMM_TILES_KS(X, 2) KTUNE_GEMM_TILES_KS(X, 4) X(8, 8, 1) X(8, 8, 2)

#define KTUNE_CONV_TILES_CS(X, CS) \
    X(1, 1, CS) X(1, 2, CS) X(1, 4, CS) X(1, 8, CS) X(1, 16, CS) \
    X(2, 1, CS) X(2, 2, CS) X(2, 4, CS) X(2, 8, CS) X(2, 16, CS) \
    X(4, 1, CS) X(4, 2, CS) X(4, 4, CS) X(4, 8, CS) X(4, 16, CS) \
    X(8, 1, CS) X(8, 2, CS) X(8, 4, CS) X(8, 8, CS)

#define KTUNE_CONV_TILES(X) KTUNE_CONV_TILES_CS(X, 1) X(8, 16, 1) KTUNE_CONV_TILES_CS(X, 2)

// NARROW (<= 256 threads, up to 255 registers) variants: the tiles whose wide
// instantiation is register-capped below 255 (accumulators <= 32).
#define KTUNE_GEMM_TILES_NARROW_KS(X, KS) \
    X(1, 1, KS) X(1, 2, KS) X(2, 1, KS) X(1, 4, KS) X(2, 2, KS) X(4, 1, KS) X(1, 8, KS) X(2, 4, KS) X(4, 2, KS) \
    X(8, 1, KS)
#define KTUNE_GEMM_TILES_NARROW(X)                                                                        \
    KTUNE_GEMM_TILES_NARROW_KS(X, 1) KTUNE_GEMM_TILES_NARROW_KS(X, 2) X(2, 8, 1) X(4, 4, 1) X(8, 2, 1) \
    X(4, 8, 1) X(8, 4, 1) X(1, 1, 4) X(1, 2, 4) X(2, 1, 4) X(1, 4, 4) X(2, 2, 4) X(4, 1, 4) X(1, 8, 4) X(2, 4, 4) \
    X(4, 2, 4) X(8, 1, 4) X(2, 8, 2) X(4, 4, 2) X(8, 2, 2)
#define KTUNE_CONV_TILES_NARROW(X)                                                                                \
    X(1, 1, 1) X(1, 2, 1) X(1, 4, 1) X(1, 8, 1) X(1, 16, 1) X(2, 1, 1) X(2, 2, 1) X(2, 4, 1) X(2, 8, 1) X(2, 16, 1) \
    X(4, 1, 1) X(4, 2, 1) X(4, 4, 1) X(4, 8, 1) X(8, 1, 1) X(8, 2, 1) X(8, 4, 1) X(1, 1, 2) X(1, 2, 2) X(1, 4, 2)  \
    X(1, 8, 2) X(1, 16, 2) X(2, 1, 2) X(2, 2, 2) X(2, 4, 2) X(2, 8, 2) X(4, 1, 2) X(4, 2, 2) X(4, 4, 2) X(8, 1, 2) \
    X(8, 2, 2)

namespace ktune_dev {

// Kernel pointer lookup per (kind, dtype, mode); defined in
// simt_<kind>_<T>_<mode>.cu.  Returns nullptr for tiles outside the envelope;
// (0,0,0) is the generic runtime-tile instantiation.
#define KTUNE_DECLARE_LOOKUP(KIND, T, MODE) const void* simt_##KIND##_##T##_##MODE(int ms, int ns, int ks);
#define KTUNE_DECLARE_GEMM_LOOKUPS(T, MODE)          \
    KTUNE_DECLARE_LOOKUP(gemm, T, MODE##_nn)         \
    KTUNE_DECLARE_LOOKUP(gemm, T, MODE##_tn)         \
    KTUNE_DECLARE_LOOKUP(gemm, T, MODE##_nt)         \
    KTUNE_DECLARE_LOOKUP(gemm, T, MODE##_tt)
KTUNE_DECLARE_GEMM_LOOKUPS(f32, parity)
KTUNE_DECLARE_GEMM_LOOKUPS(f32, fast)
KTUNE_DECLARE_GEMM_LOOKUPS(f64, parity)
KTUNE_DECLARE_GEMM_LOOKUPS(f64, fast)
KTUNE_DECLARE_LOOKUP(conv, f32, parity)
KTUNE_DECLARE_LOOKUP(conv, f32, fast)
KTUNE_DECLARE_LOOKUP(conv, f64, parity)
KTUNE_DECLARE_LOOKUP(conv, f64, fast)
KTUNE_DECLARE_GEMM_LOOKUPS(f32, parity_narrow)
KTUNE_DECLARE_GEMM_LOOKUPS(f32, fast_narrow)
KTUNE_DECLARE_LOOKUP(conv, f32, parity_narrow)
KTUNE_DECLARE_LOOKUP(conv, f32, fast_narrow)
// TMA-fed fp32 GEMM (simt_tma.cuh), NARROW tile list, no generic instantiation
const void* simt_tma_f32_parity_nn(int ms, int ns, int ks);
const void* simt_tma_f32_parity_tn(int ms, int ns, int ks);
const void* simt_tma_f32_parity_nt(int ms, int ns, int ks);
const void* simt_tma_f32_parity_tt(int ms, int ns, int ks);
const void* simt_tma_f32_fast_nn(int ms, int ns, int ks);
const void* simt_tma_f32_fast_tn(int ms, int ns, int ks);
const void* simt_tma_f32_fast_nt(int ms, int ns, int ks);
const void* simt_tma_f32_fast_tt(int ms, int ns, int ks);

// Max threads the (ms,ns,ks) instantiation was compiled for.
inline int simt_thread_cap(int ms, int ns, int ks) {
    if (ms == 0) return 1024;
    const int acc = ms * ns * ks;
    return acc <= 16 ? 1024 : (acc <= 32 ? 512 : 256);
}

}  // namespace ktune_dev
