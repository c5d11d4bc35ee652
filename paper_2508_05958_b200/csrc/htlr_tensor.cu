// Device-backed tensor building blocks of the reference's per-block API
// (htlr.tensor / htlr.blocks, tensor.py:35-132, blocks.py:126-259): mode
// products, GEMM (for contract and the low-rank baseline), Kronecker products
// and the thin Householder QR with LAPACK's conventions (dgeqr2 + dorg2r: R's
// diagonal is -sign(a_ii) * norm, the same signs numpy.linalg.qr returns).
// These serve the drop-in functions users call on single blocks; the plan's
// construction and matvec never go through them.  Host arrays in and out
// (row-major, C order), computed on the current device.
#include "htlr_device.cuh"
#include "htlr_kernels.h"

#include <algorithm>
#include <vector>

namespace htlr {

namespace {

// out[a, r, b] = sum_k m[r, k] t[a, k, b]   (t: A x K x B, m: M x K)
__global__ void mode_product_kernel(const double* __restrict__ t, const double* __restrict__ m, int64_t A, int64_t K,
                                    int64_t B, int64_t M, double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= A * M * B) return;
  const int64_t b = e % B, r = (e / B) % M, a = e / (B * M);
  double acc = 0.0;
  for (int64_t k = 0; k < K; ++k) acc = fma(m[r * K + k], t[(a * K + k) * B + b], acc);
  out[e] = acc;
}

// C = A B, row-major; 16 x 16 tiles staged in shared memory
__global__ void gemm_kernel(const double* __restrict__ A, const double* __restrict__ B, int64_t m, int64_t k,
                            int64_t n, double* __restrict__ C) {
  __shared__ double sa[16][17], sb[16][17];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t row = (int64_t)blockIdx.y * 16 + ty, col = (int64_t)blockIdx.x * 16 + tx;
  double acc = 0.0;
  for (int64_t k0 = 0; k0 < k; k0 += 16) {
    sa[ty][tx] = (row < m && k0 + tx < k) ? A[row * k + k0 + tx] : 0.0;
    sb[ty][tx] = (k0 + ty < k && col < n) ? B[(k0 + ty) * n + col] : 0.0;
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) acc = fma(sa[ty][q], sb[q][tx], acc);
    __syncthreads();
  }
  if (row < m && col < n) C[row * n + col] = acc;
}

// kron(a, b): a (ar x ac), b (br x bc) -> (ar br) x (ac bc), row-major
__global__ void kron_kernel(const double* __restrict__ a, int64_t ar, int64_t ac, const double* __restrict__ b,
                            int64_t br, int64_t bc, double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t cols = ac * bc;
  if (e >= ar * br * cols) return;
  const int64_t i = e / cols, j = e % cols;
  out[e] = a[(i / br) * ac + j / bc] * b[(i % br) * bc + j % bc];
}

// Thin Householder QR of a rows x cols matrix (rows >= cols), one CTA:
// A column-major in global scratch; dgeqr2 then dorg2r, the trailing-column
// updates spread over the threads.
__global__ void qr_kernel(double* __restrict__ A, int64_t rows, int64_t cols, double* __restrict__ tau,
                          double* __restrict__ Qc) {
  __shared__ double red[1024];
  __shared__ double s_beta, s_tau, s_scal;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int64_t i = 0; i < cols; ++i) {
    double part = 0.0;
    for (int64_t kk = i + 1 + tid; kk < rows; kk += nt) part += A[kk + rows * i] * A[kk + rows * i];
    red[tid] = part;
    __syncthreads();
    for (int s = nt / 2; s > 0; s >>= 1) {
      if (tid < s) red[tid] += red[tid + s];
      __syncthreads();
    }
    if (tid == 0) {
      const double alpha = A[i + rows * i], xnorm = sqrt(red[0]);
      if (xnorm == 0.0) {
        s_tau = 0.0;
        s_beta = alpha;
        s_scal = 1.0;
      } else {
        const double beta = -copysign(hypot(alpha, xnorm), alpha);
        s_tau = (beta - alpha) / beta;
        s_beta = beta;
        s_scal = 1.0 / (alpha - beta);
      }
      tau[i] = s_tau;
    }
    __syncthreads();
    for (int64_t kk = i + 1 + tid; kk < rows; kk += nt) A[kk + rows * i] *= s_scal;
    __syncthreads();
    if (tid == 0) A[i + rows * i] = s_beta;
    // H_i = I - tau v v^T, v = [1; A[i+1:, i]], on the trailing columns
    for (int64_t j = i + 1 + tid; j < cols; j += nt) {
      double w = A[i + rows * j];
      for (int64_t kk = i + 1; kk < rows; ++kk) w += A[kk + rows * i] * A[kk + rows * j];
      w *= s_tau;
      A[i + rows * j] -= w;
      for (int64_t kk = i + 1; kk < rows; ++kk) A[kk + rows * j] -= w * A[kk + rows * i];
    }
    __syncthreads();
  }
  // dorg2r: Q = H_1 ... H_cols applied to the first cols columns of I
  for (int64_t j = tid; j < cols; j += nt)
    for (int64_t kk = 0; kk < rows; ++kk) Qc[kk + rows * j] = (kk == j) ? 1.0 : 0.0;
  __syncthreads();
  for (int64_t i = cols - 1; i >= 0; --i) {
    for (int64_t j = i + tid; j < cols; j += nt) {
      double w = Qc[i + rows * j];
      for (int64_t kk = i + 1; kk < rows; ++kk) w += A[kk + rows * i] * Qc[kk + rows * j];
      w *= tau[i];
      Qc[i + rows * j] -= w;
      for (int64_t kk = i + 1; kk < rows; ++kk) Qc[kk + rows * j] -= w * A[kk + rows * i];
    }
    __syncthreads();
  }
}

struct Buf {
  double* p = nullptr;
  ~Buf() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t n) { return cudaMalloc(&p, std::max<size_t>(1, n) * sizeof(double)); }
};

cudaError_t up(Buf& b, const double* h, size_t n) {
  cudaError_t e = b.alloc(n);
  if (e == cudaSuccess && n) e = cudaMemcpy(b.p, h, n * sizeof(double), cudaMemcpyHostToDevice);
  return e;
}

}  // namespace

cudaError_t tensor_mode_product(const double* t, int64_t A, int64_t K, int64_t B, const double* m, int64_t M,
                                double* out) {
  Buf dt, dm, dout;
  cudaError_t e = up(dt, t, A * K * B);
  if (e == cudaSuccess) e = up(dm, m, M * K);
  if (e == cudaSuccess) e = dout.alloc(A * M * B);
  if (e != cudaSuccess) return e;
  const int64_t total = A * M * B;
  if (total > 0) mode_product_kernel<<<(unsigned)((total + 255) / 256), 256>>>(dt.p, dm.p, A, K, B, M, dout.p);
  e = cudaGetLastError();
  if (e == cudaSuccess && total) e = cudaMemcpy(out, dout.p, total * sizeof(double), cudaMemcpyDeviceToHost);
  return e;
}

cudaError_t tensor_gemm(const double* a, const double* b, int64_t m, int64_t k, int64_t n, double* c) {
  Buf da, db, dc;
  cudaError_t e = up(da, a, m * k);
  if (e == cudaSuccess) e = up(db, b, k * n);
  if (e == cudaSuccess) e = dc.alloc(m * n);
  if (e != cudaSuccess) return e;
  if (m > 0 && n > 0) gemm_kernel<<<dim3((unsigned)((n + 15) / 16), (unsigned)((m + 15) / 16)), 256>>>(da.p, db.p, m, k, n, dc.p);
  e = cudaGetLastError();
  if (e == cudaSuccess && m * n) e = cudaMemcpy(c, dc.p, m * n * sizeof(double), cudaMemcpyDeviceToHost);
  return e;
}

cudaError_t tensor_kron(const double* a, int64_t ar, int64_t ac, const double* b, int64_t br, int64_t bc,
                        double* out) {
  Buf da, db, dout;
  cudaError_t e = up(da, a, ar * ac);
  if (e == cudaSuccess) e = up(db, b, br * bc);
  const int64_t total = ar * ac * br * bc;
  if (e == cudaSuccess) e = dout.alloc(total);
  if (e != cudaSuccess) return e;
  if (total) kron_kernel<<<(unsigned)((total + 255) / 256), 256>>>(da.p, ar, ac, db.p, br, bc, dout.p);
  e = cudaGetLastError();
  if (e == cudaSuccess && total) e = cudaMemcpy(out, dout.p, total * sizeof(double), cudaMemcpyDeviceToHost);
  return e;
}

cudaError_t tensor_qr(const double* a, int64_t rows, int64_t cols, double* q, double* r) {
  // column-major copies (the reflectors run down columns)
  std::vector<double> colmajor((size_t)rows * cols);
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) colmajor[i + rows * j] = a[i * cols + j];
  Buf dA, dtau, dQ;
  cudaError_t e = up(dA, colmajor.data(), colmajor.size());
  if (e == cudaSuccess) e = dtau.alloc(cols);
  if (e == cudaSuccess) e = dQ.alloc(rows * cols);
  if (e != cudaSuccess) return e;
  if (rows && cols) qr_kernel<<<1, 256>>>(dA.p, rows, cols, dtau.p, dQ.p);
  e = cudaGetLastError();
  std::vector<double> hA((size_t)rows * cols), hQ((size_t)rows * cols);
  if (e == cudaSuccess && rows * cols) e = cudaMemcpy(hA.data(), dA.p, hA.size() * sizeof(double), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && rows * cols) e = cudaMemcpy(hQ.data(), dQ.p, hQ.size() * sizeof(double), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return e;
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) q[i * cols + j] = hQ[i + rows * j];
  for (int64_t i = 0; i < cols; ++i)
    for (int64_t j = 0; j < cols; ++j) r[i * cols + j] = (j >= i) ? hA[i + rows * j] : 0.0;
  return cudaSuccess;
}

}  // namespace htlr
