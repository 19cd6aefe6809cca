// mlp_fast.cu -- the MLP performance model as batched GEMMs (fast mode).
//
// North star: "Training and the runtime candidate sweep both run as small
// batched GEMM kernels on the GPU."  K6f (sweep) and K7f (minibatch SGD) run
// every layer as one fp64 GEMM over the whole batch (cuBLAS DGEMM, the plain
// library GEMM) plus small fused kernels for bias / ReLU / ReLU' / clipped
// update.  Same model, loss, minibatching, shuffles, global-norm clip and
// best-epoch selection as perf_model.cpp:318-423 -- but GEMM summation order,
// so results match the reference to rounding, not bit for bit.  The
// bit-identical K6 / K7 (mlp.cu) stay the parity path.
//
// Layouts: a batch of activations of width w is a column-major (w x n)
// matrix (row-major n x w: one candidate's activations contiguous); layer
// weights are row-major (out x in) = column-major (in x out), packed
// [W0 b0 W1 b1 ...] exactly as mlp.cu packs them.

#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cmath>
#include <limits>
#include <mutex>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "ktune/kernels.hpp"
#include "ktune/mlp.hpp"
#include "ktune/sampling.hpp"

namespace ktune_dev {
namespace mlpf {

void cublas_check(cublasStatus_t s, const char* what) {
    if (s != CUBLAS_STATUS_SUCCESS) throw ktune::cuda_error(std::string(what) + ": cuBLAS status " + std::to_string(int(s)));
}

cublasHandle_t handle() {
    static std::mutex mu;
    static cublasHandle_t h = nullptr;
    std::lock_guard<std::mutex> lock(mu);
    if (h == nullptr) {
        cublas_check(cublasCreate(&h), "cublasCreate");
        // fixed algorithms: deterministic results run to run
        cublas_check(cublasSetMathMode(h, CUBLAS_DEFAULT_MATH), "cublasSetMathMode");
    }
    return h;
}

// x[c, o] += b[o]; relu unless last.  Z is (out x n) column-major.
__global__ void bias_act_kernel(double* __restrict__ Z, const double* __restrict__ b, int out, std::int64_t n, int relu,
                                double* __restrict__ Zpre) {
    const std::int64_t total = n * out;
    for (std::int64_t i = std::int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += std::int64_t(gridDim.x) * blockDim.x) {
        const int o = int(i % out);
        const double z = Z[i] + b[o];
        if (Zpre) Zpre[i] = z;
        Z[i] = relu ? (z > 0.0 ? z : 0.0) : z;
    }
}

// log-features of candidates: consts (already logged) then log(2^e) of each
// tuple value (powers of two), or the raw values when log_inputs is off.
__global__ void features_kernel(const double* __restrict__ consts, int n_const, const std::int32_t* __restrict__ tuples,
                                int tuple_len, const double* __restrict__ pow2_logs, int log_inputs, std::int64_t n,
                                double* __restrict__ X) {
    const int dim = n_const + tuple_len;
    for (std::int64_t r = std::int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
         r += std::int64_t(gridDim.x) * blockDim.x) {
        double* x = X + r * dim;
        for (int i = 0; i < n_const; ++i) x[i] = consts[i];
        for (int j = 0; j < tuple_len; ++j) {
            const int v = tuples[r * tuple_len + j];
            x[n_const + j] = log_inputs ? pow2_logs[31 - __clz(v)] : double(v);
        }
    }
}

// output delta: 2/B * (pred - y), residual kept for the epoch MSE
__global__ void out_delta_kernel(const double* __restrict__ pred, const double* __restrict__ y, int B, double two_over_b,
                                 double* __restrict__ delta, double* __restrict__ err) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
        const double e = pred[b] - y[b];
        err[b] = e;
        delta[b] = two_over_b * e;
    }
}

// delta *= relu'(zpre)
__global__ void relu_back_kernel(double* __restrict__ delta, const double* __restrict__ zpre, std::int64_t total) {
    for (std::int64_t i = std::int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += std::int64_t(gridDim.x) * blockDim.x)
        if (zpre[i] <= 0.0) delta[i] = 0.0;
}

// db[o] = sum_b delta[o, b]  (delta: out x B column-major)
__global__ void bias_grad_kernel(const double* __restrict__ delta, int out, int B, double* __restrict__ db) {
    for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < out; o += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int b = 0; b < B; ++b) s += delta[std::int64_t(b) * out + o];
        db[o] = s;
    }
}

// gather rows perm[start .. start+B) of X (n x dim, row-major) and Y
__global__ void gather_kernel(const double* __restrict__ X, const double* __restrict__ Y, const int* __restrict__ perm,
                              int start, int B, int dim, double* __restrict__ Xb, double* __restrict__ Yb) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < B * dim; i += gridDim.x * blockDim.x) {
        const int b = i / dim, c = i - b * dim;
        const int row = perm[start + b];
        Xb[i] = X[std::int64_t(row) * dim + c];
        if (c == 0) Yb[b] = Y[row];
    }
}

// P -= scale * G, scale = lr * min(1, clip / ||G||) (the reference clip rule)
__global__ void update_kernel(double* __restrict__ P, const double* __restrict__ G, int n, const double* __restrict__ norm,
                              double lr, double clip) {
    const double nv = *norm;
    const double scale = nv > clip ? lr * (clip / nv) : lr;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) P[i] -= scale * G[i];
}

struct Net {
    int L;
    std::vector<int> width;  // width[0] = input dim ... width[L] = 1
    std::vector<int> woff, boff;
    int nparams;
};

Net net_of(const ktune::MlpWeights& w) {
    Net d;
    d.L = int(w.layers.size());
    d.width.push_back(w.layers[0].in);
    int off = 0;
    for (const auto& l : w.layers) {
        d.woff.push_back(off);
        off += l.in * l.out;
        d.boff.push_back(off);
        off += l.out;
        d.width.push_back(l.out);
    }
    d.nparams = off;
    return d;
}

std::vector<double> pack(const ktune::MlpWeights& w) {
    std::vector<double> p;
    for (const auto& L : w.layers) {
        p.insert(p.end(), L.w.begin(), L.w.end());
        p.insert(p.end(), L.b.begin(), L.b.end());
    }
    return p;
}

void unpack(const std::vector<double>& p, ktune::MlpWeights& w) {
    std::size_t off = 0;
    for (auto& L : w.layers) {
        std::copy(p.begin() + std::ptrdiff_t(off), p.begin() + std::ptrdiff_t(off + L.w.size()), L.w.begin());
        off += L.w.size();
        std::copy(p.begin() + std::ptrdiff_t(off), p.begin() + std::ptrdiff_t(off + L.b.size()), L.b.begin());
        off += L.b.size();
    }
}

struct DevBuf {
    double* p{nullptr};
    std::size_t n{0};
    void reserve(std::size_t elems) {
        if (elems <= n) return;
        if (p) cudaFree(p);
        p = nullptr;
        ktune::dev::check(cudaMalloc(&p, std::max<std::size_t>(elems, 1) * sizeof(double)), "cudaMalloc(mlp)");
        n = elems;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

int blocks_for(std::int64_t n) { return int(std::max<std::int64_t>(1, std::min<std::int64_t>((n + 255) / 256, 148 * 8))); }

// Forward over a batch: acts[l] (width_l x n col-major); zpre[l] for l >= 1
// when training.  Returns the device pointer of the head output (1 x n).
const double* forward(const Net& d, const double* P, const double* X, std::int64_t n, std::vector<DevBuf>& acts,
                      std::vector<DevBuf>* zpre, cudaStream_t s) {
    cublasHandle_t h = handle();
    cublas_check(cublasSetStream(h, s), "cublasSetStream");
    const double one = 1.0, zero = 0.0;
    const double* a = X;
    for (int l = 0; l < d.L; ++l) {
        const int in = d.width[std::size_t(l)], out = d.width[std::size_t(l) + 1];
        acts[std::size_t(l) + 1].reserve(std::size_t(n) * out);
        double* z = acts[std::size_t(l) + 1].p;
        // Z (out x n) = W (out x in, row-major = col-major in x out, transposed) * A (in x n)
        cublas_check(cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, out, int(n), in, &one, P + d.woff[std::size_t(l)], in, a,
                                 in, &zero, z, out),
                     "cublasDgemm(forward)");
        double* zp = nullptr;
        if (zpre) {
            (*zpre)[std::size_t(l) + 1].reserve(std::size_t(n) * out);
            zp = (*zpre)[std::size_t(l) + 1].p;
        }
        bias_act_kernel<<<blocks_for(n * out), 256, 0, s>>>(z, P + d.boff[std::size_t(l)], out, n, l + 1 < d.L ? 1 : 0,
                                                            zp);
        ktune::dev::check(cudaGetLastError(), "mlp bias launch");
        a = z;
    }
    return a;
}

}  // namespace mlpf
}  // namespace ktune_dev

namespace ktune {

using namespace ktune_dev::mlpf;

void mlp_predict_tuples_fast(const MlpWeights& w, const std::vector<double>& const_features, const std::int32_t* tuples,
                             std::int64_t n, int tuple_len, double* out, double* device_seconds) {
    w.validate();
    if (int(const_features.size()) + tuple_len != w.input_dim())
        throw std::invalid_argument("feature vector has wrong dimension");
    if (n == 0) return;
    std::vector<double> consts = const_features;
    if (w.log_inputs)
        for (double& v : consts) {
            if (!(v > 0.0)) throw std::invalid_argument("features must be strictly positive under the log transform");
            v = std::log(v);
        }
    double pow2_logs[31];
    for (int e = 0; e < 31; ++e) pow2_logs[e] = std::log(double(1u << e));
    const Net d = net_of(w);
    const std::vector<double> params = pack(w);
    // persistent per-process device buffers (grown on demand)
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    static DevBuf dP, dC, dL, dX;
    static std::vector<DevBuf> acts(kMaxMlpLayers + 1);
    static std::int32_t* dT = nullptr;
    static std::size_t dT_n = 0;
    dP.reserve(params.size());
    dC.reserve(consts.size() + 1);
    dL.reserve(31);
    dX.reserve(std::size_t(n) * std::size_t(d.width[0]));
    if (std::size_t(n) * tuple_len > dT_n) {
        if (dT) cudaFree(dT);
        dev::check(cudaMalloc(&dT, std::size_t(n) * tuple_len * 4), "cudaMalloc(tuples)");
        dT_n = std::size_t(n) * tuple_len;
    }
    if (int(acts.size()) < d.L + 1) acts.resize(std::size_t(d.L) + 1);
    cudaStream_t s = nullptr;
    dev::check(cudaMemcpyAsync(dP.p, params.data(), params.size() * 8, cudaMemcpyHostToDevice, s), "H2D params");
    dev::check(cudaMemcpyAsync(dC.p, consts.data(), consts.size() * 8, cudaMemcpyHostToDevice, s), "H2D consts");
    dev::check(cudaMemcpyAsync(dL.p, pow2_logs, sizeof(pow2_logs), cudaMemcpyHostToDevice, s), "H2D logs");
    dev::check(cudaMemcpyAsync(dT, tuples, std::size_t(n) * tuple_len * 4, cudaMemcpyHostToDevice, s), "H2D tuples");
    cudaEvent_t e0, e1;
    dev::check(cudaEventCreate(&e0), "cudaEventCreate");
    dev::check(cudaEventCreate(&e1), "cudaEventCreate");
    dev::check(cudaEventRecord(e0, s), "cudaEventRecord");
    features_kernel<<<blocks_for(n), 256, 0, s>>>(dC.p, int(consts.size()), dT, tuple_len, dL.p, w.log_inputs ? 1 : 0, n,
                                                  dX.p);
    dev::check(cudaGetLastError(), "mlp features launch");
    const double* head = forward(d, dP.p, dX.p, n, acts, nullptr, s);
    dev::check(cudaEventRecord(e1, s), "cudaEventRecord");
    dev::check(cudaMemcpyAsync(out, head, std::size_t(n) * 8, cudaMemcpyDeviceToHost, s), "D2H predictions");
    dev::check(cudaStreamSynchronize(s), "mlp sweep sync");
    float ms = 0;
    dev::check(cudaEventElapsedTime(&ms, e0, e1), "cudaEventElapsedTime");
    if (device_seconds) *device_seconds = double(ms) * 1e-3;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
}

TrainResult mlp_train_fast(const TrainingSet& train, const TrainingSet& val, const MlpArchitecture& arch,
                           const TrainConfig& cfg) {
    arch.validate();
    cfg.validate();
    train.validate();
    val.validate();
    if (train.dim != arch.input_dim || val.dim != arch.input_dim)
        throw std::invalid_argument("training data does not match architecture");
    std::mt19937_64 rng(cfg.rng_seed);
    MlpWeights w = init_weights(arch, rng());
    const Net d = net_of(w);
    const std::size_t n = train.size(), nv = val.size();
    const int dim = train.dim;
    std::vector<double> xt(train.features), xv(val.features);
    if (w.log_inputs) {
        for (double& v : xt) {
            if (!(v > 0.0)) throw std::invalid_argument("features must be strictly positive under the log transform");
            v = std::log(v);
        }
        for (double& v : xv) {
            if (!(v > 0.0)) throw std::invalid_argument("features must be strictly positive under the log transform");
            v = std::log(v);
        }
    }
    std::vector<double> params = pack(w);
    const int np = int(params.size());
    const int bs = std::min<int>(cfg.batch_size, int(n));
    DevBuf dP, dG, dX, dY, dXv, dYv, dXb, dYb, dErr, dVerr, dNorm;
    dP.reserve(std::size_t(np));
    dG.reserve(std::size_t(np));
    dX.reserve(xt.size());
    dY.reserve(n);
    dXv.reserve(std::max<std::size_t>(xv.size(), 1));
    dYv.reserve(std::max<std::size_t>(nv, 1));
    dXb.reserve(std::size_t(bs) * dim);
    dYb.reserve(std::size_t(bs));
    dErr.reserve(n);
    dVerr.reserve(std::max<std::size_t>(nv, 1));
    dNorm.reserve(1);
    std::vector<DevBuf> acts(std::size_t(d.L) + 1), zpre(std::size_t(d.L) + 1), delta(std::size_t(d.L) + 1);
    for (int l = 0; l <= d.L; ++l) delta[std::size_t(l)].reserve(std::size_t(bs) * d.width[std::size_t(l)]);
    int* dperm = nullptr;
    dev::check(cudaMalloc(&dperm, std::max<std::size_t>(n, 1) * 4), "cudaMalloc(perm)");
    cudaStream_t s = nullptr;
    dev::check(cudaMemcpy(dP.p, params.data(), np * 8, cudaMemcpyHostToDevice), "H2D params");
    dev::check(cudaMemcpy(dX.p, xt.data(), xt.size() * 8, cudaMemcpyHostToDevice), "H2D train X");
    dev::check(cudaMemcpy(dY.p, train.targets.data(), n * 8, cudaMemcpyHostToDevice), "H2D train Y");
    if (nv) {
        dev::check(cudaMemcpy(dXv.p, xv.data(), xv.size() * 8, cudaMemcpyHostToDevice), "H2D val X");
        dev::check(cudaMemcpy(dYv.p, val.targets.data(), nv * 8, cudaMemcpyHostToDevice), "H2D val Y");
    }
    cublasHandle_t h = handle();
    cublas_check(cublasSetStream(h, s), "cublasSetStream");
    const double one = 1.0, zero = 0.0;
    std::vector<int> perm(n);
    std::iota(perm.begin(), perm.end(), 0);
    std::vector<double> err(n), verr(nv);
    TrainResult result;
    result.best_val_mse = std::numeric_limits<double>::infinity();
    try {
        for (int epoch = 0; epoch < cfg.epochs; ++epoch) {
            for (std::size_t i = n; i > 1; --i) std::swap(perm[i - 1], perm[index_below(rng, i)]);
            dev::check(cudaMemcpyAsync(dperm, perm.data(), n * 4, cudaMemcpyHostToDevice, s), "H2D perm");
            for (int start = 0; start < int(n); start += cfg.batch_size) {
                const int B = std::min(cfg.batch_size, int(n) - start);
                gather_kernel<<<blocks_for(std::int64_t(B) * dim), 256, 0, s>>>(dX.p, dY.p, dperm, start, B, dim, dXb.p,
                                                                               dYb.p);
                const double* pred = forward(d, dP.p, dXb.p, B, acts, &zpre, s);
                out_delta_kernel<<<blocks_for(B), 256, 0, s>>>(pred, dYb.p, B, 2.0 / double(B), delta[std::size_t(d.L)].p,
                                                              dErr.p + start);
                for (int l = d.L - 1; l >= 0; --l) {
                    const int in = d.width[std::size_t(l)], out = d.width[std::size_t(l) + 1];
                    const double* a = l == 0 ? dXb.p : acts[std::size_t(l)].p;
                    // dW (col-major in x out) = A (in x B) * delta_l^T (B x out)
                    cublas_check(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, in, out, B, &one, a, in,
                                             delta[std::size_t(l) + 1].p, out, &zero, dG.p + d.woff[std::size_t(l)], in),
                                 "cublasDgemm(dW)");
                    bias_grad_kernel<<<blocks_for(out), 256, 0, s>>>(delta[std::size_t(l) + 1].p, out, B,
                                                                     dG.p + d.boff[std::size_t(l)]);
                    if (l > 0) {
                        // delta_{l-1} (in x B) = W (col-major in x out) * delta_l (out x B), then relu'
                        cublas_check(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, in, B, out, &one,
                                                 dP.p + d.woff[std::size_t(l)], in, delta[std::size_t(l) + 1].p, out,
                                                 &zero, delta[std::size_t(l)].p, in),
                                     "cublasDgemm(delta)");
                        relu_back_kernel<<<blocks_for(std::int64_t(B) * in), 256, 0, s>>>(
                            delta[std::size_t(l)].p, zpre[std::size_t(l)].p, std::int64_t(B) * in);
                    }
                }
                cublas_check(cublasSetPointerMode(h, CUBLAS_POINTER_MODE_DEVICE), "cublasSetPointerMode");
                cublas_check(cublasDnrm2(h, np, dG.p, 1, dNorm.p), "cublasDnrm2");
                cublas_check(cublasSetPointerMode(h, CUBLAS_POINTER_MODE_HOST), "cublasSetPointerMode");
                update_kernel<<<blocks_for(np), 256, 0, s>>>(dP.p, dG.p, np, dNorm.p, cfg.learning_rate,
                                                             cfg.clip_grad_norm);
                dev::check(cudaGetLastError(), "mlp train step launch");
            }
            // validation residuals with the updated weights
            if (nv) {
                const double* vpred = forward(d, dP.p, dXv.p, std::int64_t(nv), acts, nullptr, s);
                dev::check(cudaMemcpyAsync(verr.data(), vpred, nv * 8, cudaMemcpyDeviceToHost, s), "D2H val pred");
            }
            dev::check(cudaMemcpyAsync(err.data(), dErr.p, n * 8, cudaMemcpyDeviceToHost, s), "D2H residuals");
            dev::check(cudaStreamSynchronize(s), "mlp epoch sync");
            long double running = 0.0L, vacc = 0.0L;
            for (std::size_t i = 0; i < n; ++i) running += (long double)err[i] * err[i];
            for (std::size_t i = 0; i < nv; ++i) {
                const long double e = (long double)verr[i] - val.targets[i];
                vacc += e * e;
            }
            EpochStats st;
            st.train_mse = double(running / (long double)(n));
            st.val_mse = nv ? double(vacc / (long double)(nv)) : st.train_mse;
            result.history.push_back(st);
            if (!std::isfinite(st.val_mse))
                throw std::runtime_error("training diverged: validation MSE became non-finite at epoch " +
                                         std::to_string(epoch));
            if (st.val_mse < result.best_val_mse) {
                result.best_val_mse = st.val_mse;
                result.best_epoch = epoch;
                dev::check(cudaMemcpy(params.data(), dP.p, np * 8, cudaMemcpyDeviceToHost), "D2H params");
                unpack(params, w);
                result.weights = w;
            }
        }
    } catch (...) {
        cudaFree(dperm);
        throw;
    }
    cudaFree(dperm);
    return result;
}

}  // namespace ktune
