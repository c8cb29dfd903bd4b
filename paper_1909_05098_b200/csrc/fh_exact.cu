// EXACT mode: the reference's explicit step with its floating-point
// operation order, on the GPU.  Compiled with -fmad=false; every product and
// sum below is an explicit _rn intrinsic, so results are bit-identical to the
// numba kernels of /root/reference/pkg/src/fedheat/kernels.py (verified by
// tests/test_gpu_parity.py against the reference's golden vectors).
//
// Step = 2 launches:
//   k_exact_elem : per element, contrib[p] = kbar_e * sum_b A[a,b] (T_b - T_e0)
//                  (kernels.py:101-129; TD: kbar from k(T) of the corners,
//                  kernels.py:76-98)
//   k_exact_node : per node, the chunked sum of kernels.py:113-134 as a CSR
//                  gather (partial per 4096-element chunk, decremented in
//                  element order; partials added in chunk order), fused with
//                  the lumped update of kernels.py:137-142, the Dirichlet
//                  overwrite and the runaway check of solver.py:364-382.
#include "fh_exact_dev.cuh"

namespace fh {

__device__ __forceinline__ double elem_kbar(const ExactArgs &g, int64_t e, const double *__restrict__ T) {
  const int64_t lo = eoff(g, e), hi = eoff(g, e + 1);
  const int r = g.elem_region ? g.elem_region[e] : 0;
  const Curve<double> &kc = g.mats.m[r].k;
  double s = 0.0;
  for (int64_t p = lo; p < hi; ++p) s = add(s, interp_rn(kc, T[g.conn[p]]));
  double kb = dvd(s, (double)(hi - lo));
  if (g.kfactor) kb = mul(kb, g.kfactor[e]);
  return kb;
}

// TI freeze / explicit kbar+capacity refresh (solver.py:280-296)
__global__ void k_exact_props(ExactArgs g, const double *__restrict__ T) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < g.E) g.kbar[t] = elem_kbar(g, t, T);
  if (t < g.V) {
    const Mat<double> &m = g.mats.m[g.node_region ? g.node_region[t] : 0];
    const double x = T[t];
    g.cap[t] = mul(mul(interp_rn(m.rho, x), interp_rn(m.c, x)), g.node_vol[t]);
    if (m.td_perf) {
      const double kb = mul(mul(interp_rn(m.wb, x), m.cb), g.node_vol[t]);
      g.kb[t] = kb;
      g.qb[t] = mul(kb, m.Ta);
    }
  }
}

__global__ void k_exact_elem(ExactArgs g, const double *__restrict__ T, int use_frozen_kbar,
                             const double *__restrict__ kbar_in, unsigned long long step_no) {
  // skip only when an earlier step failed (the failing step runs to completion)
  if (g.flag && g.flag->step < step_no) return;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= g.E) return;
  const double ke = kbar_in ? kbar_in[e] : (use_frozen_kbar ? g.kbar[e] : elem_kbar(g, e, T));
  const int64_t p0 = eoff(g, e);
  const int n = (int)(eoff(g, e + 1) - p0);
  const double *__restrict__ A = g.mat + moff(g, e);
  const double t0 = T[g.conn[p0]];
  double d[8];
  for (int b = 0; b < n; ++b) d[b] = sub(T[g.conn[p0 + b]], t0);
  for (int a = 0; a < n; ++a) {
    double acc = 0.0;
    for (int b = 0; b < n; ++b) acc = add(acc, mul(A[a * n + b], d[b]));
    g.contrib[p0 + a] = mul(ke, acc);
  }
}

__device__ __forceinline__ double chunked_gather(const ExactArgs &g, int64_t i) {
  double total = 0.0, part = 0.0;
  int64_t cur = -1;
  for (int32_t q = g.csr_offs[i]; q < g.csr_offs[i + 1]; ++q) {
    const int32_t p = g.csr_pos[q];
    const int64_t chunk = elem_of_pos(g, p) / g.chunk_size;
    if (chunk != cur) {
      if (cur >= 0) total = add(total, part);
      part = 0.0;
      cur = chunk;
    }
    part = sub(part, g.contrib[p]);
  }
  if (cur >= 0) total = add(total, part);
  return total;
}

__global__ void k_exact_node(ExactArgs g, double *__restrict__ T, double dt, double t_start,
                             unsigned long long step_no, int td) {
  if (g.flag && g.flag->step < step_no) return;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  bool bad = false;
  if (i < g.V) {
    const double F = chunked_gather(g, i);
    if (g.F) g.F[i] = F;
    const double xn = exact_update(g, i, F, T[i], dt, t_start, td);
    T[i] = xn;
    bad = !isfinite(xn) || fabs(xn) > g.runaway_limit;
  }
  if (g.flag && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicMin(&g.flag->step, step_no);
}

__global__ void k_gather_probes(const double *__restrict__ T, const int32_t *__restrict__ probes, int64_t np,
                                double *__restrict__ out, const FailFlag *flag) {
  if (flag && flag->step != kNoFail) return;
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q < np) out[q] = T[probes[q]];
}

void exact_props(const ExactArgs &g, const double *T, cudaStream_t s) {
  const int64_t n = g.E > g.V ? g.E : g.V;
  k_exact_props<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(g, T);
  FH_CUDA(cudaGetLastError());
}

void exact_step(const ExactArgs &g, double *T, double dt, double t_start, int64_t step_no, bool td,
                cudaStream_t s) {
  k_exact_elem<<<(unsigned)((g.E + 255) / 256), 256, 0, s>>>(g, T, td ? 0 : 1, nullptr,
                                                              (unsigned long long)step_no);
  k_exact_node<<<(unsigned)((g.V + 255) / 256), 256, 0, s>>>(g, T, dt, t_start, (unsigned long long)step_no,
                                                              td ? 1 : 0);
  FH_CUDA(cudaGetLastError());
}

// scatter only (solver.py:223-240): contributions with a given kbar, then the gather into F
__global__ void k_exact_gather_only(ExactArgs g, double *__restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < g.V) out[i] = chunked_gather(g, i);
}

void exact_scatter(const ExactArgs &g, const double *kbar, const double *T, double *out, cudaStream_t s) {
  ExactArgs h = g;
  h.flag = nullptr;
  k_exact_elem<<<(unsigned)((g.E + 255) / 256), 256, 0, s>>>(h, T, 0, kbar, 0ull);
  k_exact_gather_only<<<(unsigned)((g.V + 255) / 256), 256, 0, s>>>(h, out);
  FH_CUDA(cudaGetLastError());
}

void gather_probes(const double *T, const int32_t *probes, int64_t np, double *out, const FailFlag *flag,
                   cudaStream_t s) {
  if (np <= 0) return;
  k_gather_probes<<<(unsigned)((np + 127) / 128), 128, 0, s>>>(T, probes, np, out, flag);
  FH_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// solver.py:384-405 Gershgorin bound, reference reduction orders:
//   kbar_e = (k_0 + (((k_1 + k_2) + ...) + k_{n-1})) / n      (np.add.reduceat)
//   row_i  = ((0 + kbar_e1*ra_1) + kbar_e2*ra_2) + ...         (np.add.at, element order)
//   lam_i  = (row_i + kb_i) / C_i over C_i > 0 ; dt = 2 / max lam
__global__ void k_crit_kbar(ExactArgs g, const double *__restrict__ T, double *__restrict__ kbar) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= g.E) return;
  const int64_t lo = eoff(g, e), hi = eoff(g, e + 1);
  const Curve<double> &kc = g.mats.m[g.elem_region ? g.elem_region[e] : 0].k;
  double rest = 0.0;
  for (int64_t p = lo + 1; p < hi; ++p) {
    const double kv = interp_rn(kc, T[g.conn[p]]);
    rest = (p == lo + 1) ? kv : add(rest, kv);
  }
  double kb = dvd(add(interp_rn(kc, T[g.conn[lo]]), rest), (double)(hi - lo));
  if (g.kfactor) kb = mul(kb, g.kfactor[e]);
  kbar[e] = kb;
}

__global__ void k_crit_node(ExactArgs g, const double *__restrict__ T, const double *__restrict__ kbar,
                            double *__restrict__ lam_out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= g.V) return;
  double row = 0.0;
  for (int32_t q = g.csr_offs[i]; q < g.csr_offs[i + 1]; ++q) {
    const int32_t p = g.csr_pos[q];
    row = add(row, mul(kbar[elem_of_pos(g, p)], g.row_abs[p]));
  }
  const Mat<double> &m = g.mats.m[g.node_region ? g.node_region[i] : 0];
  const double x = T[i], v = g.node_vol[i];
  const double kb = m.td_perf ? mul(mul(interp_rn(m.wb, x), m.cb), v) : g.kb[i];
  row = add(row, kb);
  if (g.robin_slot && g.robin_slot[i] >= 0) row = add(row, g.robin_hA[g.robin_slot[i]]);
  const double cap = mul(mul(interp_rn(m.rho, x), interp_rn(m.c, x)), v);
  lam_out[i] = cap > 0.0 ? dvd(row, cap) : -INFINITY;
}

void exact_critical(const ExactArgs &g, const double *T, double *kbar_scratch, double *lam, cudaStream_t s) {
  k_crit_kbar<<<(unsigned)((g.E + 255) / 256), 256, 0, s>>>(g, T, kbar_scratch);
  k_crit_node<<<(unsigned)((g.V + 255) / 256), 256, 0, s>>>(g, T, kbar_scratch, lam);
  FH_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// operator layer kernels (kernels.py:76-142)
__global__ void k_op_curve(Curve<double> c, const double *__restrict__ T, int64_t n, double *__restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = interp_rn(c, T[i]);
}
__global__ void k_op_capacity(Curve<double> r, Curve<double> c, const double *__restrict__ T,
                              const double *__restrict__ v, int64_t n, double *__restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = mul(mul(interp_rn(r, T[i]), interp_rn(c, T[i])), v[i]);
}
__global__ void k_op_mean(const int32_t *__restrict__ conn, const int64_t *__restrict__ offs, int64_t E,
                          const double *__restrict__ nodal, double *__restrict__ out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= E) return;
  double s = 0.0;
  for (int64_t p = offs[e]; p < offs[e + 1]; ++p) s = add(s, nodal[conn[p]]);
  out[e] = dvd(s, (double)(offs[e + 1] - offs[e]));
}
__global__ void k_op_update(double *__restrict__ T, const double *__restrict__ F, const double *__restrict__ C,
                            const double *__restrict__ kb, const double *__restrict__ qb,
                            const double *__restrict__ qm, const double *__restrict__ qr, int64_t n, double dt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = T[i];
  const double rate = add(add(add(sub(F[i], mul(kb[i], x)), qb[i]), qm[i]), qr[i]);
  T[i] = add(x, dvd(mul(dt, rate), C[i]));
}

void op_curve(const Curve<double> &c, const double *T, int64_t n, double *out, cudaStream_t s) {
  k_op_curve<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(c, T, n, out);
  FH_CUDA(cudaGetLastError());
}
void op_capacity(const Curve<double> &r, const Curve<double> &c, const double *T, const double *v, int64_t n,
                 double *out, cudaStream_t s) {
  k_op_capacity<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(r, c, T, v, n, out);
  FH_CUDA(cudaGetLastError());
}
void op_mean(const int32_t *conn, const int64_t *offs, int64_t E, const double *nodal, double *out,
             cudaStream_t s) {
  k_op_mean<<<(unsigned)((E + 255) / 256), 256, 0, s>>>(conn, offs, E, nodal, out);
  FH_CUDA(cudaGetLastError());
}
void op_update(double *T, const double *F, const double *C, const double *kb, const double *qb, const double *qm,
               const double *qr, int64_t n, double dt, cudaStream_t s) {
  k_op_update<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(T, F, C, kb, qb, qm, qr, n, dt);
  FH_CUDA(cudaGetLastError());
}

}  // namespace fh
