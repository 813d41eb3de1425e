// Per-op device kernels on reference-layout (NCHW fp32) tensors: the ops::
// surface of /root/reference/proj/include/denseplan/ops.hpp, one kernel per
// reference function.  These back the dpb_op_* C-ABI entry points used for
// op-level parity; the fused block path (dpb_block.cu) does not call them.
#include <cuda_runtime.h>

#include "dpb_common.cuh"

namespace dpb {

// Block-wide fixed-order fp64 reduction of two values (256 threads).
__device__ __forceinline__ void block_sum2(double& a, double& b) {
  __shared__ double sa[8], sb[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  const int w = threadIdx.x / 32;
  if (threadIdx.x % 32 == 0) { sa[w] = a; sb[w] = b; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0;
    for (int i = 0; i < 8; ++i) { x += sa[i]; y += sb[i]; }
    sa[0] = x;
    sb[0] = y;
  }
  __syncthreads();
  a = sa[0];
  b = sb[0];
  __syncthreads();
}

// batch_statistics, ops.hpp:138-162: one CTA per channel.
__global__ void __launch_bounds__(256)
op_batch_statistics(const float* __restrict__ x, int64_t n, int64_t c, int64_t hw,
                    float* __restrict__ mean, float* __restrict__ var) {
  const int64_t ch = blockIdx.x;
  double s1 = 0.0, s2 = 0.0;
  for (int64_t i = threadIdx.x; i < n * hw; i += blockDim.x) {
    const int64_t img = i / hw, p = i - img * hw;
    const double v = x[(img * c + ch) * hw + p];
    s1 += v;
    s2 += v * v;
  }
  block_sum2(s1, s2);
  if (threadIdx.x == 0) {
    const double cnt = static_cast<double>(n * hw);
    const double m = s1 / cnt;
    double v = s2 / cnt - m * m;
    mean[ch] = static_cast<float>(m);
    var[ch] = static_cast<float>(v < 0.0 ? 0.0 : v);
  }
}

// batchnorm_apply (+ optional relu_inplace), ops.hpp:115-134, 261-264.
__global__ void op_batchnorm_apply(const float* __restrict__ x, int64_t n, int64_t c,
                                   int64_t hw, const float* __restrict__ gamma,
                                   const float* __restrict__ beta,
                                   const float* __restrict__ mean,
                                   const float* __restrict__ var, int relu,
                                   float* __restrict__ dst) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n * c * hw) return;
  const int64_t ch = (i / hw) % c;
  const float inv = bn_inv(var[ch]);
  float y = gamma[ch] * (x[i] - mean[ch]) * inv + beta[ch];
  if (relu) y = y > 0.f ? y : 0.f;
  dst[i] = y;
}

// batchnorm_backward, ops.hpp:206-243: one CTA per channel, two passes.
__global__ void __launch_bounds__(256)
op_batchnorm_backward(const float* __restrict__ gy, const float* __restrict__ x, int64_t n,
                      int64_t c, int64_t hw, const float* __restrict__ gamma,
                      const float* __restrict__ mean, const float* __restrict__ var,
                      float* __restrict__ gx, float* __restrict__ dgamma,
                      float* __restrict__ dbeta) {
  const int64_t ch = blockIdx.x;
  const float mu = mean[ch];
  const float inv = bn_inv(var[ch]);
  double sg = 0.0, sgx = 0.0;
  for (int64_t i = threadIdx.x; i < n * hw; i += blockDim.x) {
    const int64_t img = i / hw, p = i - img * hw;
    const int64_t o = (img * c + ch) * hw + p;
    const float g = gy[o];
    const float xh = (x[o] - mu) * inv;
    sg += g;
    sgx += static_cast<double>(g) * xh;
  }
  block_sum2(sg, sgx);
  const double cnt = static_cast<double>(n * hw);
  const float mg = static_cast<float>(sg / cnt), mgx = static_cast<float>(sgx / cnt);
  if (threadIdx.x == 0) {
    dgamma[ch] = static_cast<float>(sgx);
    dbeta[ch] = static_cast<float>(sg);
  }
  const float gi = gamma[ch] * inv;
  for (int64_t i = threadIdx.x; i < n * hw; i += blockDim.x) {
    const int64_t img = i / hw, p = i - img * hw;
    const int64_t o = (img * c + ch) * hw + p;
    const float xh = (x[o] - mu) * inv;
    gx[o] = gi * (gy[o] - mg - xh * mgx);
  }
}

// conv2d_forward (stride 1), ops.hpp:315-342: one thread per output.
__global__ void op_conv2d_forward(const float* __restrict__ x, int64_t n, int64_t cin,
                                  int64_t h, int64_t w, const float* __restrict__ wt,
                                  int64_t cout, int kk, int pad, float* __restrict__ dst) {
  const int64_t oh = h + 2 * pad - kk + 1, ow = w + 2 * pad - kk + 1;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n * cout * oh * ow) return;
  const int64_t ox = i % ow, oy = (i / ow) % oh, oc = (i / (ow * oh)) % cout,
                img = i / (ow * oh * cout);
  float acc = 0.f;
  for (int64_t ic = 0; ic < cin; ++ic)
    for (int ky = 0; ky < kk; ++ky) {
      const int64_t iy = oy - pad + ky;
      if (iy < 0 || iy >= h) continue;
      for (int kx = 0; kx < kk; ++kx) {
        const int64_t ix = ox - pad + kx;
        if (ix < 0 || ix >= w) continue;
        acc = fmaf(x[((img * cin + ic) * h + iy) * w + ix],
                   wt[((oc * cin + ic) * kk + ky) * kk + kx], acc);
      }
    }
  dst[i] = acc;
}

// conv2d_backward dgrad (gather form), ops.hpp:346-387: thread per input elem.
__global__ void op_conv2d_dgrad(const float* __restrict__ gy, int64_t n, int64_t cin,
                                int64_t h, int64_t w, const float* __restrict__ wt,
                                int64_t cout, int kk, int pad, float* __restrict__ gx) {
  const int64_t oh = h + 2 * pad - kk + 1, ow = w + 2 * pad - kk + 1;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n * cin * h * w) return;
  const int64_t ix = i % w, iy = (i / w) % h, ic = (i / (w * h)) % cin, img = i / (w * h * cin);
  float acc = 0.f;
  for (int64_t oc = 0; oc < cout; ++oc)
    for (int ky = 0; ky < kk; ++ky) {
      const int64_t oy = iy + pad - ky;
      if (oy < 0 || oy >= oh) continue;
      for (int kx = 0; kx < kk; ++kx) {
        const int64_t ox = ix + pad - kx;
        if (ox < 0 || ox >= ow) continue;
        acc = fmaf(gy[((img * cout + oc) * oh + oy) * ow + ox],
                   wt[((oc * cin + ic) * kk + ky) * kk + kx], acc);
      }
    }
  gx[i] = acc;
}

// conv2d_backward wgrad: one CTA per weight element, fp64 reduction.
__global__ void __launch_bounds__(256)
op_conv2d_wgrad(const float* __restrict__ gy, const float* __restrict__ x, int64_t n,
                int64_t cin, int64_t h, int64_t w, int64_t cout, int kk, int pad,
                float* __restrict__ gw) {
  const int64_t oh = h + 2 * pad - kk + 1, ow = w + 2 * pad - kk + 1;
  const int64_t widx = blockIdx.x;
  const int kx = static_cast<int>(widx % kk), ky = static_cast<int>((widx / kk) % kk);
  const int64_t ic = (widx / (kk * kk)) % cin, oc = widx / (kk * kk * cin);
  double s = 0.0, unused = 0.0;
  for (int64_t i = threadIdx.x; i < n * oh * ow; i += blockDim.x) {
    const int64_t img = i / (oh * ow), oy = (i / ow) % oh, ox = i % ow;
    const int64_t iy = oy - pad + ky, ix = ox - pad + kx;
    if (iy < 0 || iy >= h || ix < 0 || ix >= w) continue;
    s += static_cast<double>(gy[((img * cout + oc) * oh + oy) * ow + ox]) *
         x[((img * cin + ic) * h + iy) * w + ix];
  }
  block_sum2(s, unused);
  if (threadIdx.x == 0) gw[widx] = static_cast<float>(s);
}

// relu_forward / relu_inplace, ops.hpp:248-264 (v > 0 ? v : 0; dst may be x).
__global__ void op_relu_forward(const float* x, int64_t count, float* dst) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < count) {
    const float v = x[i];
    dst[i] = v > 0.f ? v : 0.f;
  }
}

// relu_backward(_inplace), ops.hpp:268-287: grad_x = ref > 0 ? grad_y : 0
// (subgradient 0 at 0; ref may be the ReLU input or output).
__global__ void op_relu_backward(const float* gy, const float* __restrict__ ref, int64_t count, float* gx) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < count) gx[i] = ref[i] > 0.f ? gy[i] : 0.f;
}

static unsigned nblk(int64_t n) { return static_cast<unsigned>((n + 255) / 256); }

int op_relu_forward(const float* x, int64_t count, float* dst, cudaStream_t st) {
  if (count > 0) op_relu_forward<<<nblk(count), 256, 0, st>>>(x, count, dst);
  return cudaGetLastError();
}
int op_relu_backward(const float* gy, const float* ref, int64_t count, float* gx, cudaStream_t st) {
  if (count > 0) op_relu_backward<<<nblk(count), 256, 0, st>>>(gy, ref, count, gx);
  return cudaGetLastError();
}

// concat_forward / concat_backward, ops.hpp:53-107: per sample, input i's
// c_i*h*w contiguous values go to channels [off_i, off_i + c_i) of the NCHW
// destination (copy_into, tensor.hpp:168-180) — strided device copies, no
// arithmetic.  backward copies the channel slices back out.
int op_concat(int count, const float* const* parts, const int64_t* channels, int64_t n, int64_t hw, float* whole,
              int64_t whole_c, int backward, cudaStream_t st) {
  int64_t off = 0;
  for (int i = 0; i < count; ++i) {
    const size_t run = static_cast<size_t>(channels[i] * hw) * sizeof(float);
    float* slot = whole + off * hw;
    const size_t wp = static_cast<size_t>(whole_c * hw) * sizeof(float);
    const cudaError_t e =
        backward ? cudaMemcpy2DAsync(const_cast<float*>(parts[i]), run, slot, wp, run, static_cast<size_t>(n),
                                     cudaMemcpyDeviceToDevice, st)
                 : cudaMemcpy2DAsync(slot, wp, parts[i], run, run, static_cast<size_t>(n), cudaMemcpyDeviceToDevice,
                                     st);
    if (e != cudaSuccess) return e;
    off += channels[i];
  }
  return cudaSuccess;
}

int op_batch_statistics(const float* x, int64_t n, int64_t c, int64_t h, int64_t w,
                        float* mean, float* var, cudaStream_t st) {
  op_batch_statistics<<<static_cast<unsigned>(c), 256, 0, st>>>(x, n, c, h * w, mean, var);
  return cudaGetLastError();
}
int op_batchnorm_apply(const float* x, int64_t n, int64_t c, int64_t h, int64_t w,
                       const float* g, const float* b, const float* mean, const float* var,
                       int relu, float* dst, cudaStream_t st) {
  op_batchnorm_apply<<<nblk(n * c * h * w), 256, 0, st>>>(x, n, c, h * w, g, b, mean, var,
                                                           relu, dst);
  return cudaGetLastError();
}
int op_batchnorm_backward(const float* gy, const float* x, int64_t n, int64_t c, int64_t h,
                          int64_t w, const float* g, const float* mean, const float* var,
                          float* gx, float* dg, float* db, cudaStream_t st) {
  op_batchnorm_backward<<<static_cast<unsigned>(c), 256, 0, st>>>(gy, x, n, c, h * w, g, mean,
                                                                  var, gx, dg, db);
  return cudaGetLastError();
}
int op_conv2d_forward(const float* x, int64_t n, int64_t cin, int64_t h, int64_t w,
                      const float* wt, int64_t cout, int kk, int pad, float* dst,
                      cudaStream_t st) {
  const int64_t oh = h + 2 * pad - kk + 1, ow = w + 2 * pad - kk + 1;
  op_conv2d_forward<<<nblk(n * cout * oh * ow), 256, 0, st>>>(x, n, cin, h, w, wt, cout, kk,
                                                                pad, dst);
  return cudaGetLastError();
}
int op_conv2d_backward(const float* gy, const float* x, int64_t n, int64_t cin, int64_t h,
                       int64_t w, const float* wt, int64_t cout, int kk, int pad, float* gx,
                       float* gw, cudaStream_t st) {
  if (gx) op_conv2d_dgrad<<<nblk(n * cin * h * w), 256, 0, st>>>(gy, n, cin, h, w, wt, cout, kk,
                                                                 pad, gx);
  op_conv2d_wgrad<<<static_cast<unsigned>(cout * cin * kk * kk), 256, 0, st>>>(
      gy, x, n, cin, h, w, cout, kk, pad, gw);
  return cudaGetLastError();
}

}  // namespace dpb
