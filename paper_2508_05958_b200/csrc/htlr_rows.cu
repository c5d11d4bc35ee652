// Exact rows of the Nystrom system on the device: the reference's
// exact_row_evaluator (oracles.py:65-100) behind estimate_rel_error_random
// (operators.py:216-239), i.e. SURVEY 8(f) row f2.
//   out[r] = sum_{j != i} k(x_i, x_j) w_j u_j + (diag_i + a_i) u_i,  i = rows[r]
// uniform grid: w_j = h^d, diag_i = h^d * cell average (kernels.py:252-265);
// mapped grid : w_j = product of cell widths, diag_i = cell integral.
// Kernel values use the reference formula (kernel_from_r2).  One CTA per row,
// deterministic block reduction.
#include "htlr_kernels.h"

namespace htlr {

__global__ void exact_rows_kernel(KernelParams kp, int d, int n, double h, double hd, const double* __restrict__ coords,
                                  const double* __restrict__ widths, const int64_t* __restrict__ rows,
                                  const double* __restrict__ diag_rows, const double* __restrict__ avec,
                                  double aconst, const double* __restrict__ u, double* __restrict__ out) {
  __shared__ double red[256];
  const int64_t i = rows[blockIdx.x];
  const int64_t N = (d == 2) ? (int64_t)n * n : (int64_t)n * n * n;
  int ii[3] = {(int)(i % n), (int)((i / n) % n), d == 3 ? (int)(i / ((int64_t)n * n)) : 0};
  double x[3];
  for (int a = 0; a < d; ++a) x[a] = coords ? coords[ii[a]] : __dmul_rn(__dadd_rn((double)ii[a], 0.5), h);
  double acc = 0.0;
  for (int64_t j = threadIdx.x; j < N; j += blockDim.x) {
    if (j == i) continue;
    int jj[3] = {(int)(j % n), (int)((j / n) % n), d == 3 ? (int)(j / ((int64_t)n * n)) : 0};
    double y[3];
    double w = coords ? 1.0 : hd;
    for (int a = 0; a < d; ++a) {
      y[a] = coords ? coords[jj[a]] : __dmul_rn(__dadd_rn((double)jj[a], 0.5), h);
      if (coords) w = w * widths[jj[a]];
    }
    acc += kernel_from_r2(kp, r2_of(d, x, y)) * w * u[j];
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double a = avec ? avec[i] : aconst;
    out[blockIdx.x] = red[0] + (diag_rows[blockIdx.x] + a) * u[i];
  }
}

// per-row diagonal: uniform -> h^d * cell average; mapped -> cell integral
__global__ void row_diag_kernel(int d, int n, double hd, const double* __restrict__ cell_avg,
                                const double* __restrict__ dvec_all, const int64_t* __restrict__ rows, int64_t nrows,
                                double* __restrict__ out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  out[r] = dvec_all ? dvec_all[rows[r]] : cell_avg[0] * hd;
}

void launch_exact_rows(const KernelParams& kp, int d, int n, double h, double hd, const double* coords,
                       const double* widths, const int64_t* rows, int64_t nrows, const double* cell_avg,
                       const double* dvec_all, double* diag_rows, const double* avec, double aconst,
                       const double* u, double* out, cudaStream_t st) {
  if (nrows <= 0) return;
  row_diag_kernel<<<(unsigned)((nrows + 255) / 256), 256, 0, st>>>(d, n, hd, cell_avg, dvec_all, rows, nrows,
                                                                   diag_rows);
  exact_rows_kernel<<<(unsigned)nrows, 256, 0, st>>>(kp, d, n, h, hd, coords, widths, rows, diag_rows, avec, aconst,
                                                     u, out);
}

}  // namespace htlr
