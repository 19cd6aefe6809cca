// mlp.cu -- K6 (candidate sweep) and K7 (minibatch SGD) of the MLP
// performance model, fp64 on the GPU.
//
// K6 reproduces MlpModel::predict_batch (perf_model.cpp:429-450) bit for bit:
// each output accumulates bias + a[i]*w[o,i] in input order with separately
// rounded multiply and add (the reference is built without FMA), relu on
// hidden layers, linear head.  Log-features come from glibc on the host (or
// from host-built tables of log(2^e) for tuple values), never from the
// device log().
//
// K7 runs one epoch per launch on one CTA, minibatch by minibatch, keeping
// the reference's operation order (perf_model.cpp:121-197, 303-314): per
// weight the gradient sums rows in order (skipping zero deltas), deltas sum
// output units in order, the update is w - scale*g.  The only deviation is
// the global-norm clip (double instead of x87 long double), which changes a
// step only when the norm exceeds clip_grad_norm.  Shuffles, train/val MSE
// (summed on the host in long double) and best-epoch selection follow
// perf_model.cpp:318-397 exactly.

#include <cuda_runtime.h>

#include <cmath>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "ktune/kernels.hpp"
#include "ktune/mlp.hpp"
#include "ktune/sampling.hpp"

namespace ktune_dev {
namespace mlp {

constexpr int kMaxLayers = 8;

struct Dims {
    int L;                       // layers (hidden + head)
    int width[kMaxLayers + 1];   // width[0] = input dim, width[L] = 1
    int woff[kMaxLayers];        // offset of layer l weights in the packed params
    int boff[kMaxLayers];        // offset of layer l bias
    int aoff[kMaxLayers + 1];    // offset of activation l in a row's activation record
    int act_len;                 // sum of widths (activation record length)
    int nparams;
};

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }

// Forward of one row.  a: input (log-features), len width[0].  If rec is
// non-null, the whole activation record (inputs, relu'd hidden activations)
// and the pre-activations are stored for backprop.
template <int MAXW>
__device__ double forward_row(const double* __restrict__ P, const Dims& d, const double* x, double* rec, double* zrec) {
    double a[MAXW], z[MAXW];
    for (int i = 0; i < d.width[0]; ++i) a[i] = x[i];
    if (rec)
        for (int i = 0; i < d.width[0]; ++i) rec[i] = a[i];
    for (int l = 0; l < d.L; ++l) {
        const int in = d.width[l], out = d.width[l + 1];
        const double* w = P + d.woff[l];
        const double* b = P + d.boff[l];
        for (int o = 0; o < out; ++o) {
            double acc = __ldg(b + o);
            const double* wr = w + o * in;
            for (int i = 0; i < in; ++i) acc = add(acc, mul(a[i], __ldg(wr + i)));
            z[o] = acc;
        }
        if (zrec)
            for (int o = 0; o < out; ++o) zrec[d.aoff[l + 1] + o] = z[o];
        if (l + 1 < d.L) {
            for (int o = 0; o < out; ++o) a[o] = z[o] > 0.0 ? z[o] : 0.0;
            if (rec)
                for (int o = 0; o < out; ++o) rec[d.aoff[l + 1] + o] = a[o];
        }
    }
    return z[0];
}

template <int MAXW>
__global__ void sweep_kernel(const double* __restrict__ P, const Dims d, const double* __restrict__ const_logs,
                             int n_const, const std::int32_t* __restrict__ tuples, int tuple_len,
                             const double* __restrict__ pow2_logs, int log_inputs, std::int64_t n,
                             double* __restrict__ out) {
    double x[MAXW];
    for (std::int64_t r = std::int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
         r += std::int64_t(gridDim.x) * blockDim.x) {
        for (int i = 0; i < n_const; ++i) x[i] = const_logs[i];
        const std::int32_t* t = tuples + r * tuple_len;
        for (int j = 0; j < tuple_len; ++j) {
            const int v = t[j];
            x[n_const + j] = log_inputs ? pow2_logs[31 - __clz(v)] : double(v);
        }
        out[r] = forward_row<MAXW>(P, d, x, nullptr, nullptr);
    }
}

template <int MAXW>
__global__ void rows_kernel(const double* __restrict__ P, const Dims d, const double* __restrict__ X, std::int64_t n,
                            double* __restrict__ out) {
    for (std::int64_t r = std::int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
         r += std::int64_t(gridDim.x) * blockDim.x)
        out[r] = forward_row<MAXW>(P, d, X + r * d.width[0], nullptr, nullptr);
}

// Validation residuals e = pred - y (the host squares and sums them in long double).
template <int MAXW>
__global__ void residual_kernel(const double* __restrict__ P, const Dims d, const double* __restrict__ X,
                                const double* __restrict__ Y, std::int64_t n, double* __restrict__ err) {
    for (std::int64_t r = std::int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
         r += std::int64_t(gridDim.x) * blockDim.x)
        err[r] = forward_row<MAXW>(P, d, X + r * d.width[0], nullptr, nullptr) - Y[r];
}

constexpr int kTrainThreads = 256;

// One epoch of minibatch SGD on one CTA.
template <int MAXW>
__global__ void __launch_bounds__(kTrainThreads) train_epoch_kernel(
    double* __restrict__ P, double* __restrict__ G, const double* __restrict__ X, const double* __restrict__ Y,
    const int* __restrict__ perm, int n, int batch, const Dims d, double lr, double clip, double* __restrict__ acts,
    double* __restrict__ zs, double* __restrict__ deltas, double* __restrict__ row_err) {
    __shared__ double red[kTrainThreads];
    const int tid = threadIdx.x;
    const int T = blockDim.x;
    const int L = d.L;
    const int A = d.act_len;
    for (int start = 0; start < n; start += batch) {
        const int B = min(batch, n - start);
        const double two_over_b = 2.0 / double(B);
        // ---- forward, residuals, output delta
        for (int b = tid; b < B; b += T) {
            const int row = perm[start + b];
            const double pred = forward_row<MAXW>(P, d, X + std::int64_t(row) * d.width[0], acts + std::int64_t(b) * A,
                                                  zs + std::int64_t(b) * A);
            const double y = Y[row];
            row_err[start + b] = pred - y;
            deltas[std::int64_t(b) * A + d.aoff[L]] = mul(two_over_b, pred - y);
        }
        __syncthreads();
        // ---- backward
        for (int l = L - 1; l >= 0; --l) {
            const int in = d.width[l], out = d.width[l + 1];
            // gradient of layer l: rows summed in order, zero deltas skipped
            for (int idx = tid; idx < out * in + out; idx += T) {
                double g = 0.0;
                if (idx < out * in) {
                    const int o = idx / in, i = idx - o * in;
                    for (int b = 0; b < B; ++b) {
                        const double dl = deltas[std::int64_t(b) * A + d.aoff[l + 1] + o];
                        if (dl == 0.0) continue;
                        g = add(g, mul(dl, acts[std::int64_t(b) * A + d.aoff[l] + i]));
                    }
                    G[d.woff[l] + idx] = g;
                } else {
                    const int o = idx - out * in;
                    for (int b = 0; b < B; ++b) {
                        const double dl = deltas[std::int64_t(b) * A + d.aoff[l + 1] + o];
                        if (dl == 0.0) continue;
                        g = add(g, dl);
                    }
                    G[d.boff[l] + o] = g;
                }
            }
            if (l > 0) {
                // delta_{l-1}[b,i] = relu'(z) * sum_o delta_l[b,o] * w[o,i] (o in order)
                const double* w = P + d.woff[l];
                for (int b = tid; b < B; b += T) {
                    const double* dl = deltas + std::int64_t(b) * A + d.aoff[l + 1];
                    double* dp = deltas + std::int64_t(b) * A + d.aoff[l];
                    const double* zp = zs + std::int64_t(b) * A + d.aoff[l];
                    for (int i = 0; i < in; ++i) {
                        double p = 0.0;
                        for (int o = 0; o < out; ++o) {
                            if (dl[o] == 0.0) continue;
                            p = add(p, mul(dl[o], w[o * in + i]));
                        }
                        dp[i] = zp[i] <= 0.0 ? 0.0 : p;
                    }
                }
            }
            __syncthreads();
        }
        // ---- global-norm clip and update
        double s = 0.0;
        for (int i = tid; i < d.nparams; i += T) s = fma(G[i], G[i], s);
        red[tid] = s;
        __syncthreads();
        for (int stride = T / 2; stride > 0; stride >>= 1) {
            if (tid < stride) red[tid] += red[tid + stride];
            __syncthreads();
        }
        const double norm = sqrt(red[0]);
        double scale = lr;
        if (norm > clip) scale = mul(scale, clip / norm);
        for (int i = tid; i < d.nparams; i += T) P[i] = __dsub_rn(P[i], mul(scale, G[i]));
        __syncthreads();
    }
}

Dims make_dims(const ktune::MlpWeights& w) {
    Dims d{};
    d.L = int(w.layers.size());
    if (d.L > kMaxLayers) throw std::invalid_argument("mlp has more layers than the GPU kernels support (8)");
    d.width[0] = w.layers[0].in;
    int off = 0;
    for (int l = 0; l < d.L; ++l) {
        d.width[l + 1] = w.layers[std::size_t(l)].out;
        d.woff[l] = off;
        off += d.width[l] * d.width[l + 1];
        d.boff[l] = off;
        off += d.width[l + 1];
    }
    d.nparams = off;
    int a = 0;
    for (int l = 0; l <= d.L; ++l) {
        d.aoff[l] = a;
        a += d.width[l];
    }
    d.act_len = a;
    return d;
}

int max_width(const Dims& d) {
    int m = 0;
    for (int l = 0; l <= d.L; ++l) m = std::max(m, d.width[l]);
    return m;
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

struct Buf {
    void* p{nullptr};
    explicit Buf(std::size_t bytes) { ktune::dev::check(cudaMalloc(&p, std::max<std::size_t>(bytes, 16)), "cudaMalloc"); }
    ~Buf() {
        if (p) cudaFree(p);
    }
    Buf(const Buf&) = delete;
    Buf& operator=(const Buf&) = delete;
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

int grid_for(std::int64_t n, int threads) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return int(std::max<std::int64_t>(1, std::min<std::int64_t>((n + threads - 1) / threads, std::int64_t(sms) * 16)));
}

#define KTUNE_MLP_DISPATCH(MW, CALL)                                                     \
    do {                                                                                 \
        if ((MW) <= 64) {                                                                \
            constexpr int W_ = 64;                                                       \
            CALL;                                                                        \
        } else if ((MW) <= 512) {                                                        \
            constexpr int W_ = 512;                                                      \
            CALL;                                                                        \
        } else {                                                                         \
            throw std::invalid_argument("mlp layer wider than 512 units is not supported on the GPU"); \
        }                                                                                \
    } while (0)

}  // namespace mlp
}  // namespace ktune_dev

namespace ktune {

using namespace ktune_dev::mlp;

namespace {

void log_matrix(const MlpWeights& w, const double* x, std::size_t n, int dim, std::vector<double>& out) {
    out.assign(x, x + n * std::size_t(dim));
    if (!w.log_inputs) return;
    for (double& v : out) {
        if (!(v > 0.0)) throw std::invalid_argument("features must be strictly positive under the log transform");
        v = std::log(v);
    }
}

}  // namespace

void MlpModel::predict_batch(const std::vector<std::vector<double>>& rows, std::vector<double>& out) const {
    weights.validate();
    out.resize(rows.size());
    if (rows.empty()) return;
    const int dim = weights.input_dim();
    std::vector<double> flat;
    flat.reserve(rows.size() * std::size_t(dim));
    for (const auto& r : rows) {
        if (int(r.size()) != dim) throw std::invalid_argument("feature vector has wrong dimension");
        flat.insert(flat.end(), r.begin(), r.end());
    }
    std::vector<double> x;
    log_matrix(weights, flat.data(), rows.size(), dim, x);
    const Dims d = make_dims(weights);
    const std::vector<double> params = pack(weights);
    Buf dp(params.size() * 8), dx(x.size() * 8), dout(rows.size() * 8);
    dev::check(cudaMemcpy(dp.p, params.data(), params.size() * 8, cudaMemcpyHostToDevice), "H2D params");
    dev::check(cudaMemcpy(dx.p, x.data(), x.size() * 8, cudaMemcpyHostToDevice), "H2D features");
    const std::int64_t n = std::int64_t(rows.size());
    KTUNE_MLP_DISPATCH(max_width(d), (rows_kernel<W_><<<grid_for(n, 128), 128>>>(dp.as<double>(), d, dx.as<double>(),
                                                                                 n, dout.as<double>())));
    dev::check(cudaGetLastError(), "mlp rows launch");
    dev::check(cudaMemcpy(out.data(), dout.p, rows.size() * 8, cudaMemcpyDeviceToHost), "D2H predictions");
}

void mlp_predict_tuples(const MlpWeights& w, const std::vector<double>& const_features, const std::int32_t* tuples,
                        std::int64_t n, int tuple_len, double* out) {
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
    for (int e = 0; e < 31; ++e) pow2_logs[e] = std::log(double(1u << e));  // glibc, as the reference
    const Dims d = make_dims(w);
    const std::vector<double> params = pack(w);
    Buf dp(params.size() * 8), dc(consts.size() * 8 + 8), dt(std::size_t(n) * tuple_len * 4), dl(sizeof(pow2_logs)),
        dout(std::size_t(n) * 8);
    dev::check(cudaMemcpy(dp.p, params.data(), params.size() * 8, cudaMemcpyHostToDevice), "H2D params");
    dev::check(cudaMemcpy(dc.p, consts.data(), consts.size() * 8, cudaMemcpyHostToDevice), "H2D consts");
    dev::check(cudaMemcpy(dt.p, tuples, std::size_t(n) * tuple_len * 4, cudaMemcpyHostToDevice), "H2D tuples");
    dev::check(cudaMemcpy(dl.p, pow2_logs, sizeof(pow2_logs), cudaMemcpyHostToDevice), "H2D log table");
    KTUNE_MLP_DISPATCH(max_width(d),
                       (sweep_kernel<W_><<<grid_for(n, 128), 128>>>(dp.as<double>(), d, dc.as<double>(),
                                                                   int(consts.size()), dt.as<std::int32_t>(), tuple_len,
                                                                   dl.as<double>(), w.log_inputs ? 1 : 0, n,
                                                                   dout.as<double>())));
    dev::check(cudaGetLastError(), "mlp sweep launch");
    dev::check(cudaMemcpy(out, dout.p, std::size_t(n) * 8, cudaMemcpyDeviceToHost), "D2H predictions");
}

TrainResult mlp_train(const TrainingSet& train, const TrainingSet& val, const MlpArchitecture& arch,
                      const TrainConfig& cfg) {
    if (cfg.fast) return mlp_train_fast(train, val, arch, cfg);
    arch.validate();
    cfg.validate();
    train.validate();
    val.validate();
    if (train.dim != arch.input_dim || val.dim != arch.input_dim)
        throw std::invalid_argument("training data does not match architecture");
    std::mt19937_64 rng(cfg.rng_seed);
    MlpWeights w = init_weights(arch, rng());
    const Dims d = make_dims(w);
    const int mw = max_width(d);
    const std::size_t n = train.size(), nv = val.size();
    std::vector<double> xt, xv;
    log_matrix(w, train.features.data(), n, train.dim, xt);
    log_matrix(w, val.features.data(), nv, val.dim, xv);
    std::vector<double> params = pack(w);
    const std::size_t np = params.size();
    const int bs = std::min<int>(cfg.batch_size, int(n));
    Buf dP(np * 8), dG(np * 8), dX(xt.size() * 8), dY(n * 8), dXv(xv.size() * 8), dYv(nv * 8), dperm(n * 4),
        dacts(std::size_t(bs) * d.act_len * 8), dzs(std::size_t(bs) * d.act_len * 8),
        ddel(std::size_t(bs) * d.act_len * 8), derr(n * 8), dverr(nv * 8);
    dev::check(cudaMemcpy(dP.p, params.data(), np * 8, cudaMemcpyHostToDevice), "H2D params");
    dev::check(cudaMemcpy(dX.p, xt.data(), xt.size() * 8, cudaMemcpyHostToDevice), "H2D train X");
    dev::check(cudaMemcpy(dY.p, train.targets.data(), n * 8, cudaMemcpyHostToDevice), "H2D train Y");
    dev::check(cudaMemcpy(dXv.p, xv.data(), xv.size() * 8, cudaMemcpyHostToDevice), "H2D val X");
    dev::check(cudaMemcpy(dYv.p, val.targets.data(), nv * 8, cudaMemcpyHostToDevice), "H2D val Y");
    std::vector<int> perm(n);
    std::iota(perm.begin(), perm.end(), 0);
    std::vector<double> err(n), verr(nv);
    TrainResult result;
    result.best_val_mse = std::numeric_limits<double>::infinity();
    for (int epoch = 0; epoch < cfg.epochs; ++epoch) {
        for (std::size_t i = n; i > 1; --i) std::swap(perm[i - 1], perm[index_below(rng, i)]);
        dev::check(cudaMemcpy(dperm.p, perm.data(), n * 4, cudaMemcpyHostToDevice), "H2D perm");
        KTUNE_MLP_DISPATCH(mw, (train_epoch_kernel<W_><<<1, kTrainThreads>>>(
                                   dP.as<double>(), dG.as<double>(), dX.as<double>(), dY.as<double>(), dperm.as<int>(),
                                   int(n), cfg.batch_size, d, cfg.learning_rate, cfg.clip_grad_norm, dacts.as<double>(),
                                   dzs.as<double>(), ddel.as<double>(), derr.as<double>())));
        dev::check(cudaGetLastError(), "mlp train launch");
        KTUNE_MLP_DISPATCH(mw, (residual_kernel<W_><<<grid_for(std::int64_t(nv), 128), 128>>>(
                                   dP.as<double>(), d, dXv.as<double>(), dYv.as<double>(), std::int64_t(nv),
                                   dverr.as<double>())));
        dev::check(cudaMemcpy(err.data(), derr.p, n * 8, cudaMemcpyDeviceToHost), "D2H residuals");
        dev::check(cudaMemcpy(verr.data(), dverr.p, nv * 8, cudaMemcpyDeviceToHost), "D2H val residuals");
        long double running = 0.0L, vacc = 0.0L;
        for (std::size_t i = 0; i < n; ++i) {
            const long double e = err[i];
            running += e * e;
        }
        for (std::size_t i = 0; i < nv; ++i) {
            const long double e = verr[i];
            vacc += e * e;
        }
        EpochStats st;
        st.train_mse = double(running / (long double)(n));
        st.val_mse = double(vacc / (long double)(nv));
        result.history.push_back(st);
        if (!std::isfinite(st.val_mse))
            throw std::runtime_error("training diverged: validation MSE became non-finite at epoch " +
                                     std::to_string(epoch) + " (lr=" + std::to_string(cfg.learning_rate) +
                                     ", batch=" + std::to_string(cfg.batch_size) + ")");
        if (st.val_mse < result.best_val_mse) {
            result.best_val_mse = st.val_mse;
            result.best_epoch = epoch;
            dev::check(cudaMemcpy(params.data(), dP.p, np * 8, cudaMemcpyDeviceToHost), "D2H params");
            unpack(params, w);
            result.weights = w;
        }
    }
    return result;
}

}  // namespace ktune
