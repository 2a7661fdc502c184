#include <atomic>
// train.cu — training-step kernels: losses and the optimizer update.
//
// Replaces tensor.mse / softmax_cross_entropy (tensor.py:368-400), optim.adam_step
// (optim.py:31-54) and sgd_step (18-21).  Losses reduce deterministically (fixed-order fp64
// tree); the optimizer runs on one flat fp32 buffer (all parameters of the model), which is
// also the buffer the data-parallel step all-reduces.
#include "common.cuh"

namespace ukan {

// per-row CE loss (fp64) and gradient
__global__ void xent_rows_kernel(const float* __restrict__ logits, const int64_t* __restrict__ labels,
                                 double* __restrict__ row_loss, float* __restrict__ dlogits,
                                 int64_t n, int c, double gscale_over_n, int32_t* __restrict__ err) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const float* z = logits + (size_t)r * c;
  const int64_t lab = labels[r];
  float* dz = dlogits + (size_t)r * c;
  if (lab < 0 || lab >= c) {  // the reference indexes logp[rows, labels] and raises IndexError
    row_loss[r] = NAN;        // (tensor.py:388-392): flag it (read_loss raises), never read OOB
    for (int j = 0; j < c; ++j) dz[j] = 0.f;
    if (err) atomicOr(err, 2);
    return;
  }
  double mx = -INFINITY;
  for (int j = 0; j < c; ++j) mx = fmax(mx, (double)z[j]);
  double se = 0.0;
  for (int j = 0; j < c; ++j) se += exp((double)z[j] - mx);
  const double lse = log(se);
  row_loss[r] = -(((double)z[lab] - mx) - lse);
  for (int j = 0; j < c; ++j) {
    double p = exp(((double)z[j] - mx) - lse);
    if (j == lab) p -= 1.0;
    dz[j] = (float)(gscale_over_n * p);
  }
}

// Squared errors summed per 256-element block in a fixed tree order (deterministic), so the final
// single-CTA sum reads n / 256 partials instead of n.
__global__ void __launch_bounds__(256) mse_rows_kernel(const float* __restrict__ pred, const float* __restrict__ target,
                                                       double* __restrict__ sq, float* __restrict__ dpred, int64_t n,
                                                       double two_over_n) {
  __shared__ double sm[256];
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double d = 0.0;
  if (t < n) {
    d = (double)pred[t] - (double)target[t];
    dpred[t] = (float)(two_over_n * d);
  }
  sm[threadIdx.x] = d * d;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) sq[blockIdx.x] = sm[0];
}

// Deterministic single-CTA sum of v[0..n) scaled by `scale` into *out.
__global__ void __launch_bounds__(1024) sum_f64_kernel(const double* __restrict__ v, int64_t n,
                                                      double scale, double* __restrict__ out) {
  __shared__ double sm[1024];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += v[i];
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sm[threadIdx.x] += sm[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sm[0] * scale;
}

__global__ void adam_kernel(float* __restrict__ p, const float* __restrict__ g,
                            float* __restrict__ m, float* __restrict__ v, int64_t n, double lr,
                            double b1, double b2, double eps, double wd, double bc1, double bc2,
                            const double* __restrict__ guard) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  if (guard && !isfinite(*guard)) return;
  const double pv = (double)p[t];
  double gv = (double)g[t];
  if (wd != 0.0) gv = gv + wd * pv;  // coupled L2 (optim.py:42-43)
  const double mv = b1 * (double)m[t] + (1.0 - b1) * gv;
  const double vv = b2 * (double)v[t] + (1.0 - b2) * gv * gv;
  m[t] = (float)mv;
  v[t] = (float)vv;
  p[t] = (float)(pv - lr * (mv / bc1) / (sqrt(vv / bc2) + eps));
}

// Graph-replayable Adam: the step counter, learning rate and bias corrections live on the device
// (a captured CUDA graph replays the same launch parameters every step).
__global__ void adam_count_kernel(int64_t* __restrict__ t, double b1, double b2, double* __restrict__ bc,
                                  const double* __restrict__ guard) {
  if (guard && !isfinite(*guard)) return;  // skipped step: the reference raises before state.t += 1
  const int64_t tt = t[0] + 1;
  t[0] = tt;
  bc[0] = 1.0 - pow(b1, (double)tt);  // optim.py:38-39
  bc[1] = 1.0 - pow(b2, (double)tt);
}

__global__ void adam_dev_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                                float* __restrict__ v, int64_t n, const double* __restrict__ lr_dev, double b1,
                                double b2, double eps, double wd, const double* __restrict__ bc,
                                const double* __restrict__ guard) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  if (guard && !isfinite(*guard)) return;
  const double lr = *lr_dev, bc1 = bc[0], bc2 = bc[1];
  const double pv = (double)p[t];
  double gv = (double)g[t];
  if (wd != 0.0) gv = gv + wd * pv;  // coupled L2 (optim.py:42-43)
  const double mv = b1 * (double)m[t] + (1.0 - b1) * gv;
  const double vv = b2 * (double)v[t] + (1.0 - b2) * gv * gv;
  m[t] = (float)mv;
  v[t] = (float)vv;
  p[t] = (float)(pv - lr * (mv / bc1) / (sqrt(vv / bc2) + eps));
}

__global__ void sgd_kernel(float* __restrict__ p, const float* __restrict__ g, int64_t n, double lr,
                           const double* __restrict__ guard) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (guard && !isfinite(*guard)) return;
  if (t < n) p[t] = (float)((double)p[t] - lr * (double)g[t]);
}

__global__ void fill_kernel(float* __restrict__ p, int64_t n, float v) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) p[t] = v;
}

}  // namespace ukan

using namespace ukan;

static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

extern "C" int ukan_softmax_xent(const float* logits, const int64_t* labels, double* loss,
                                 float* dlogits, int64_t n, int64_t c, int64_t n_global,
                                 double grad_scale, int32_t* err_flag, void* stream) {
  if (n < 1 || c < 1 || n_global < 1 || !logits || !labels || !loss || !dlogits) return UKAN_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  double* rows = reinterpret_cast<double*>(loss) + 1;  // caller provides loss[1 + n] doubles
  xent_rows_kernel<<<nblk(n, 256), 256, 0, st>>>(logits, labels, rows, dlogits, n, (int)c,
                                                  grad_scale / (double)n_global, err_flag);
  UKAN_LAUNCH_CHECK();
  sum_f64_kernel<<<1, 1024, 0, st>>>(rows, n, 1.0 / (double)n_global, loss);
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

extern "C" int ukan_mse(const float* pred, const float* target, double* loss, float* dpred,
                        int64_t n, int64_t n_global, void* stream) {
  if (n < 1 || n_global < 1 || !pred || !target || !loss || !dpred) return UKAN_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  double* rows = loss + 1;  // caller provides loss[1 + n] doubles
  mse_rows_kernel<<<nblk(n, 256), 256, 0, st>>>(pred, target, rows, dpred, n, 2.0 / (double)n_global);
  UKAN_LAUNCH_CHECK();
  sum_f64_kernel<<<1, 1024, 0, st>>>(rows, nblk(n, 256), 1.0 / (double)n_global, loss);
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

extern "C" int ukan_adam_step(float* p, const float* g, float* m, float* v, int64_t n, double lr,
                              double beta1, double beta2, double eps, double weight_decay,
                              int64_t t, const double* guard, void* stream) {
  if (n < 0 || t < 1 || !p || !g || !m || !v) return UKAN_E_ARG;
  if (n == 0) return UKAN_OK;
  const double bc1 = 1.0 - pow(beta1, (double)t);  // optim.py:38-39
  const double bc2 = 1.0 - pow(beta2, (double)t);
  adam_kernel<<<nblk(n, 256), 256, 0, (cudaStream_t)stream>>>(p, g, m, v, n, lr, beta1, beta2, eps,
                                                              weight_decay, bc1, bc2, guard);
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

extern "C" int ukan_adam_step_dev(float* p, const float* g, float* m, float* v, int64_t n, const double* lr,
                                  double beta1, double beta2, double eps, double weight_decay, int64_t* t,
                                  double* bc, const double* guard, void* stream) {
  if (n < 0 || !p || !g || !m || !v || !lr || !t || !bc) return UKAN_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  adam_count_kernel<<<1, 1, 0, st>>>(t, beta1, beta2, bc, guard);
  UKAN_LAUNCH_CHECK();
  if (n == 0) return UKAN_OK;
  adam_dev_kernel<<<nblk(n, 256), 256, 0, st>>>(p, g, m, v, n, lr, beta1, beta2, eps, weight_decay, bc, guard);
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

extern "C" int ukan_sgd_step(float* p, const float* g, int64_t n, double lr, const double* guard,
                             void* stream) {
  if (n < 0 || !p || !g) return UKAN_E_ARG;
  if (n == 0) return UKAN_OK;
  sgd_kernel<<<nblk(n, 256), 256, 0, (cudaStream_t)stream>>>(p, g, n, lr, guard);
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

extern "C" int ukan_fill_f32(float* p, int64_t n, float value, void* stream) {
  if (n < 0 || !p) return UKAN_E_ARG;
  if (n == 0) return UKAN_OK;
  fill_kernel<<<nblk(n, 256), 256, 0, (cudaStream_t)stream>>>(p, n, value);
  UKAN_LAUNCH_CHECK();
  return UKAN_OK;
}

extern "C" int ukan_version(void) { return 100; }

namespace ukan {
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t st) {
  static const bool once = [] {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    return true;
  }();
  (void)once;
  return cudaMallocAsync(p, bytes, st);
}
}  // namespace ukan

static std::atomic<int64_t> g_launches{0};
extern "C" void ukan_note_launch(void) { g_launches.fetch_add(1, std::memory_order_relaxed); }
extern "C" int64_t ukan_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

extern "C" int ukan_basis_matrix(int k, double* M_out) { return ukan_basis_matrix_impl(k, M_out); }
