// Quasi-uniform (triangle mesh) front end on the device:
//   overlap areas of triangles with uniform cells  quasi.py:123-171,222-243
//   CSR SpMV of the transfer matrices               quasi.py:174-261, 311-313
// The pipeline is T (A (S u)) with A the HTLR operator on the auxiliary grid.
#include "htlr_kernels.h"

namespace htlr {

namespace {

// Sutherland-Hodgman step against one axis-aligned half plane, in the
// reference's vertex order (quasi.py:123-140): for each edge (prev, cur)
// emit the crossing point, then cur if it is inside.
__device__ int clip_halfplane(const double* px, const double* py, int m, int axis, double bound, bool keep_le,
                              double* qx, double* qy) {
  int k = 0;
  for (int i = 0; i < m; ++i) {
    const int ip = (i == 0) ? m - 1 : i - 1;
    const double pa = axis == 0 ? px[ip] : py[ip];
    const double ca = axis == 0 ? px[i] : py[i];
    const bool prev_in = keep_le ? (pa <= bound) : (pa >= bound);
    const bool cur_in = keep_le ? (ca <= bound) : (ca >= bound);
    if (cur_in != prev_in) {
      const double t = (bound - pa) / (ca - pa);
      qx[k] = px[ip] + t * (px[i] - px[ip]);
      qy[k] = py[ip] + t * (py[i] - py[ip]);
      ++k;
    }
    if (cur_in) {
      qx[k] = px[i];
      qy[k] = py[i];
      ++k;
    }
  }
  return k;
}

}  // namespace

// one thread per (triangle, cell) candidate: area of their intersection
__global__ void overlap_kernel(const double* __restrict__ tri_xy, const int* __restrict__ cand, int64_t ncand,
                               int m_side, double* __restrict__ areas) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncand) return;
  const int t = cand[3 * c], ci = cand[3 * c + 1], cj = cand[3 * c + 2];
  const double h = 1.0 / (double)m_side;
  const double x0 = ci * h, y0 = cj * h, x1 = (ci + 1) * h, y1 = (cj + 1) * h;
  double ax[8], ay[8], bx[8], by[8];
  for (int v = 0; v < 3; ++v) {
    ax[v] = tri_xy[6 * (int64_t)t + 2 * v];
    ay[v] = tri_xy[6 * (int64_t)t + 2 * v + 1];
  }
  int m = 3;
  m = clip_halfplane(ax, ay, m, 0, x0, false, bx, by);
  if (m) m = clip_halfplane(bx, by, m, 0, x1, true, ax, ay);
  if (m) m = clip_halfplane(ax, ay, m, 1, y0, false, bx, by);
  if (m) m = clip_halfplane(bx, by, m, 1, y1, true, ax, ay);
  double area = 0.0;
  if (m >= 3) {
    double total = 0.0;
    for (int i = 0; i < m; ++i) {
      const int ip = (i == 0) ? m - 1 : i - 1;
      total += ax[ip] * ay[i] - ax[i] * ay[ip];
    }
    area = 0.5 * fabs(total);
  }
  areas[c] = area;
}

// one warp per row
__global__ void csr_spmv_kernel(const int64_t* __restrict__ rowptr, const int* __restrict__ cols,
                                const double* __restrict__ vals, int64_t nrows, const double* __restrict__ x,
                                double* __restrict__ y) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= nrows) return;
  double acc = 0.0;
  for (int64_t e = rowptr[row] + lane; e < rowptr[row + 1]; e += 32) acc += vals[e] * x[cols[e]];
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
  if (lane == 0) y[row] = acc;
}

void launch_overlap(const double* tri_xy, const int* cand, int64_t ncand, int m_side, double* areas,
                    cudaStream_t st) {
  if (ncand > 0) overlap_kernel<<<(unsigned)((ncand + 127) / 128), 128, 0, st>>>(tri_xy, cand, ncand, m_side, areas);
}

void launch_csr_spmv(const int64_t* rowptr, const int* cols, const double* vals, int64_t nrows, const double* x,
                     double* y, cudaStream_t st) {
  if (nrows > 0) csr_spmv_kernel<<<(unsigned)((nrows * 32 + 255) / 256), 256, 0, st>>>(rowptr, cols, vals, nrows, x, y);
}

}  // namespace htlr
