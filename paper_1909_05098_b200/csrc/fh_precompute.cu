// Device precompute of the constant per-element / per-node quantities
// (north_star subsystem (i)).  Compiled with -fmad=false and written with
// explicit _rn intrinsics: the arithmetic is the reference's operation order
// (/root/reference/pkg/src/fedheat/element.py:69-171, solver.py:71-76,
// mesh.py:128-150), so A, row_abs, element volumes and lumped node volumes
// come out bit-identical to the reference's numpy precompute.
#include <climits>

#include "fh_internal.h"

namespace fh {

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// element.py:69-96 cofactor inverse
__device__ double inv3(const double m[9], double inv[9]) {
  const double a = m[0], b = m[1], c = m[2], d = m[3], e = m[4], f = m[5], g = m[6], h = m[7], i = m[8];
  const double ca = sub(mul(e, i), mul(f, h));
  const double cb = sub(mul(f, g), mul(d, i));
  const double cc = sub(mul(d, h), mul(e, g));
  const double det = add(add(mul(a, ca), mul(b, cb)), mul(c, cc));
  const double adj[9] = {ca, sub(mul(c, h), mul(b, i)), sub(mul(b, f), mul(c, e)),
                         cb, sub(mul(a, i), mul(c, g)), sub(mul(c, d), mul(a, f)),
                         cc, sub(mul(b, g), mul(a, h)), sub(mul(a, e), mul(b, d))};
#pragma unroll
  for (int k = 0; k < 9; ++k) inv[k] = __ddiv_rn(adj[k], det);
  return det;
}

__constant__ double kHexSign[8][3] = {{-1, -1, -1}, {1, -1, -1}, {1, 1, -1}, {-1, 1, -1},
                                      {-1, -1, 1},  {1, -1, 1},  {1, 1, 1},  {-1, 1, 1}};

template <int N>
__device__ void element_geometry(const double *__restrict__ xyz, const int32_t *__restrict__ ids, int64_t e,
                                 int64_t pos0, int64_t mat0, const GeomOut &out) {
  double x[N][3];
#pragma unroll
  for (int a = 0; a < N; ++a)
#pragma unroll
    for (int r = 0; r < 3; ++r) x[a][r] = xyz[3 * (int64_t)ids[a] + r];
  double inv[9], det, w;
  double B[3][N];
  if constexpr (N == 4) {
    double jt[9];  // swapaxes(edges): jt[r][c] = x[c+1][r] - x[0][r]
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) jt[r * 3 + c] = sub(x[c + 1][r], x[0][r]);
    det = inv3(jt, inv);
#pragma unroll
    for (int r = 0; r < 3; ++r) {
#pragma unroll
      for (int a = 1; a < N; ++a) B[r][a] = inv[(a - 1) * 3 + r];
      B[r][0] = -add(add(B[r][1], B[r][2]), B[r][3]);
    }
    w = __ddiv_rn(det, 6.0);
  } else {
    double jac[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) s = add(s, mul(x[k][r], kHexSign[k][c] * 0.125));
        jac[r * 3 + c] = s;
      }
    det = inv3(jac, inv);
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int a = 0; a < N; ++a) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) s = add(s, mul(inv[k * 3 + r], kHexSign[a][k] * 0.125));
        B[r][a] = s;
      }
    w = mul(8.0, det);
  }
  if (!(det > 0.0)) atomicMin(out.bad, (int)e);
  out.vol[e] = w;
  if (out.A || out.row_abs) {
    double *A = out.A ? out.A + mat0 : nullptr;
#pragma unroll
    for (int r = 0; r < N; ++r) {
      double t[N];
#pragma unroll
      for (int s = 0; s < N; ++s) {
        const double v = mul(add(add(mul(B[0][r], B[0][s]), mul(B[1][r], B[1][s])), mul(B[2][r], B[2][s])), w);
        if (A) A[r * N + s] = v;
        t[s] = fabs(v);
      }
      double ra;
      if constexpr (N == 8)  // numpy pairwise_sum for a block of 8
        ra = add(add(add(t[0], t[1]), add(t[2], t[3])), add(add(t[4], t[5]), add(t[6], t[7])));
      else
        ra = add(add(add(t[0], t[1]), t[2]), t[3]);
      out.row_abs[pos0 + r] = ra;
    }
  }
  if (out.G) {
    // G = w * inv * inv^T (only used by the fast path; order irrelevant)
    double g[6];
    int q = 0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = i; j < 3; ++j) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) s += inv[i * 3 + k] * inv[j * 3 + k];
        g[q++] = s * w;
      }
#pragma unroll
    for (int k = 0; k < 6; ++k) out.G[6 * e + k] = g[k];
  }
}

__global__ void k_geometry(const double *__restrict__ xyz, const int32_t *__restrict__ conn, int64_t n_tet,
                           int64_t n_hex, GeomOut out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n_tet + n_hex) return;
  if (e < n_tet) {
    element_geometry<4>(xyz, conn + 4 * e, e, 4 * e, 16 * e, out);
  } else {
    const int64_t h = e - n_tet;
    element_geometry<8>(xyz, conn + 4 * n_tet + 8 * h, e, 4 * n_tet + 8 * h, 16 * n_tet + 64 * h, out);
  }
}

void launch_geometry(const double *xyz, const int32_t *conn, int64_t n_tet, int64_t n_hex, GeomOut out,
                     cudaStream_t s) {
  const int64_t E = n_tet + n_hex;
  if (!E) return;
  k_geometry<<<(unsigned)((E + 127) / 128), 128, 0, s>>>(xyz, conn, n_tet, n_hex, out);
  FH_CUDA(cudaGetLastError());
}

// mesh.py:128-150: shares V_e / n_e of every incident element, added from
// 0.0 in ascending value order (order independent of the element order).
constexpr int kMaxDegree = 192;

__global__ void k_node_volumes(const int32_t *__restrict__ offs, const int32_t *__restrict__ pos, int64_t V,
                               int64_t n_tet, const double *__restrict__ vol, double *__restrict__ out,
                               int *__restrict__ overflow) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= V) return;
  const int lo = offs[i], hi = offs[i + 1];
  const int d = hi - lo;
  if (d > kMaxDegree) {
    atomicMax(overflow, d);
    return;
  }
  double s[kMaxDegree];
  for (int q = 0; q < d; ++q) {
    const int64_t p = pos[lo + q];
    double share;
    if (p < 4 * n_tet) {
      share = __ddiv_rn(vol[p / 4], 4.0);
    } else {
      share = __ddiv_rn(vol[n_tet + (p - 4 * n_tet) / 8], 8.0);
    }
    int k = q;  // insertion sort ascending
    while (k > 0 && s[k - 1] > share) {
      s[k] = s[k - 1];
      --k;
    }
    s[k] = share;
  }
  double acc = 0.0;
  for (int q = 0; q < d; ++q) acc = __dadd_rn(acc, s[q]);
  out[i] = acc;
}

void launch_node_volumes(const int32_t *csr_offs, const int32_t *csr_pos, int64_t V, int64_t n_tet,
                         const double *vol, double *node_vol, cudaStream_t s) {
  int *d_over = nullptr;
  FH_CUDA(cudaMalloc(&d_over, sizeof(int)));
  FH_CUDA(cudaMemsetAsync(d_over, 0, sizeof(int), s));
  k_node_volumes<<<(unsigned)((V + 127) / 128), 128, 0, s>>>(csr_offs, csr_pos, V, n_tet, vol, node_vol, d_over);
  FH_CUDA(cudaGetLastError());
  int over = 0;
  FH_CUDA(cudaMemcpyAsync(&over, d_over, sizeof(int), cudaMemcpyDeviceToHost, s));
  FH_CUDA(cudaStreamSynchronize(s));
  cudaFree(d_over);
  if (over) fail(FH_ERR_CONFIG, "a node touches " + std::to_string(over) + " elements (limit " +
                                    std::to_string(kMaxDegree) + ")");
}

}  // namespace fh
