// Resident small-mesh path of the EXACT step: many steps per launch.
//
// On small meshes (cfg1/cfg2: 8 000 hexes, 9 261 nodes) one explicit step is a
// few microseconds of work, so the two launches per step of the EXACT path
// (k_exact_elem + k_exact_node) cost more than the step itself.  Here one
// cooperative launch runs a whole segment of steps (solver.py:468-493, the
// reference's stepping loop):
//
//   * every CTA owns a contiguous node range; its incidences (the node-sorted
//     CSR of conn positions: the same lists k_exact_node gathers) and their A
//     rows are copied into shared memory once per launch;
//   * per step: stage T (and k(T)) of the owned nodes and their halo from the
//     current buffer (L2), compute every incidence's contribution
//     kbar_e * sum_b A[a,b] (T_b - T_e0) (kernels.py:101-129), reduce each
//     owned node's incidences in chunk order (kernels.py:113-134), run the
//     lumped update, the Dirichlet overwrite and the runaway check
//     (kernels.py:137-142, solver.py:354-382) and write the other buffer;
//   * between steps the CTAs synchronise either through a grid barrier
//     (SYNC_BARRIER: every CTA then reads the fail flag, so the failing step
//     completes and nothing after it runs) or -- the default -- not at all:
//     every new temperature is published as two 8-byte words that each carry
//     half of the value and the step's stamp, and a CTA starts its next step
//     as soon as the stamped values of ITS halo nodes have arrived
//     (SYNC_STAMPED: one L2 round trip per step instead of a release / arrive /
//     poll / reload chain).  A runaway is then only recorded; the host replays
//     the launch up to the failing step (deterministic), which leaves the
//     field right after that step like the two-launch path.
//
// The arithmetic is the EXACT path's (fh_exact_dev.cuh, -fmad=false, explicit
// _rn intrinsics in the reference's order), so the fields are bit-identical
// to the two-launch path and to the reference.
#include "fh_exact_dev.cuh"
#include "fh_resident.h"

#include <algorithm>

namespace fh {

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Grid barrier on a monotonic 64-bit word (zeroed before the launch): each
// CTA adds 1 (plus kFailBit when one of its nodes ran away this step) with
// release semantics and waits (acquire) until the low bits count every CTA of
// this step.  The word it then reads holds every CTA's addition, so all CTAs
// agree on whether the step failed without another round trip.  bar.sync on
// both sides orders the CTA's other threads' global stores / loads around
// thread 0's release / acquire.
constexpr unsigned long long kFailBit = 1ull << 40;

__device__ __forceinline__ bool grid_barrier(unsigned long long *bar, unsigned long long target, bool fail,
                                             unsigned long long *s_word) {
  __syncthreads();
  if (threadIdx.x == 0) {
    red_release_add_u64(bar, 1ull + (fail ? kFailBit : 0ull));
    unsigned long long v;
    do {
      v = ld_acquire_u64(bar);
    } while ((v & (kFailBit - 1)) < target);
    *s_word = v;
  }
  __syncthreads();
  return (*s_word >> 40) != 0;
}

// Stamped words (the LL idea of collective libraries): 8-byte stores are single
// copy atomic, so {32 value bits, 32 stamp bits} arrives whole; a double is two
// such words and is complete when both carry the expected stamp.  The stamps
// of a launch are stamp0 + (steps taken in it) and never repeat across
// launches (the host hands out stamp0 from a 32-bit epoch and clears the
// buffers before it wraps), so a stale word is never mistaken for a new one.
__device__ __forceinline__ void st_stamped(unsigned long long *slot, double x, uint32_t stamp) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  const unsigned long long hi = (unsigned long long)stamp << 32;
  const unsigned long long w0 = (b & 0xffffffffull) | hi, w1 = (b >> 32) | hi;
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(slot), "l"(w0), "l"(w1) : "memory");
}
// spins until both words carry `stamp`.  Gives up (false) after ~2^22 polls or
// as soon as another CTA gave up (*lost != 0): the launch then ends and the
// host reports an internal error instead of hanging the device.
__device__ __forceinline__ bool ld_stamped(const unsigned long long *slot, uint32_t stamp, double &x,
                                           unsigned long long *lost) {
  for (int spin = 1; spin <= (1 << 22); ++spin) {
    unsigned long long w0, w1;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(slot) : "memory");
    if ((uint32_t)(w0 >> 32) == stamp && (uint32_t)(w1 >> 32) == stamp) {
      x = __longlong_as_double((long long)((w0 & 0xffffffffull) | (w1 << 32)));
      return true;
    }
    if ((spin & 1023) == 0 && *reinterpret_cast<volatile unsigned long long *>(lost) != 0ull) break;
  }
  atomicExch(lost, 1ull);
  return false;
}

template <bool TD, bool KSTAGE, bool STAMPED>
__global__ void __launch_bounds__(kResThreads, 1) k_resident(const __grid_constant__ ResidentArgs r) {
  const ExactArgs &g = r.g;
  // an earlier call's step failed: every later launch is a no-op (fh_step semantics)
  if (g.flag->step < (unsigned long long)r.step0 + 1ull) return;
  extern __shared__ __align__(16) unsigned char sm[];
  double *sT = reinterpret_cast<double *>(sm);
  double *sK = reinterpret_cast<double *>(sm + r.off_K);
  double *sA = reinterpret_cast<double *>(sm + r.off_A);
  double *sC = reinterpret_cast<double *>(sm + r.off_C);
  double *sKb = reinterpret_cast<double *>(sm + r.off_Kb);
  NodeIn *sN = reinterpret_cast<NodeIn *>(sm + r.off_N);
  uint16_t *sL = reinterpret_cast<uint16_t *>(sm + r.off_L);
  int32_t *sE = reinterpret_cast<int32_t *>(sm + r.off_E);
  int32_t *sO = reinterpret_cast<int32_t *>(sm + r.off_O);
  uint8_t *sI = sm + r.off_I;
  int32_t *sH = reinterpret_cast<int32_t *>(sm + r.off_H);
  __shared__ unsigned long long s_word;
  __shared__ int s_bad;

  const int c = blockIdx.x, tid = threadIdx.x, bd = blockDim.x;
  const int n0 = r.cta_node[c], nown = r.cta_node[c + 1] - n0;
  const int h0 = r.cta_halo[c], nh = r.cta_halo[c + 1] - h0, nloc = nown + nh;
  const int q0 = r.cta_inc[c], nq = r.cta_inc[c + 1] - q0;
  FH_DEV_CHECK(n0 >= 0 && n0 + nown <= g.V && q0 == g.csr_offs[n0], "resident CTA ranges");

  // once per launch: the incidences' A rows, local corner nodes, elements and
  // (TI) frozen kbar; the halo ids; the owned nodes' update operands and
  // incidence ranges
  for (int q = tid; q < nq; q += bd) {
    const int e = r.inc_elem[q0 + q];
    const uint8_t info = r.inc_info[q0 + q];
    const int a = info & 7, n = (info & 8) ? 8 : 4;
    const double *A = g.mat + moff(g, e) + a * n;
#pragma unroll
    for (int b = 0; b < 8; ++b) sA[8 * q + b] = b < n ? A[b] : 0.0;
    const uint4 w = reinterpret_cast<const uint4 *>(r.inc_lconn)[q0 + q];
    reinterpret_cast<uint4 *>(sL)[q] = w;
    sE[q] = e;
    sI[q] = info;
    if (!TD) sKb[q] = g.kbar[e];
  }
  for (int i = tid; i < nh; i += bd) sH[i] = r.halo_nodes[h0 + i];
  for (int i = tid; i < nown; i += bd) sN[i] = load_node(g, n0 + i, TD ? 1 : 0);
  for (int i = tid; i <= nown; i += bd) sO[i] = g.csr_offs[n0 + i] - q0;
  if (tid == 0) s_bad = 0;
  __syncthreads();

  const Curve<double> &k0 = g.mats.m[0].k;
  int64_t done = r.nsteps;
  if (STAMPED) {
    // publish the owned nodes of the field as given (stamp of step 0 of this launch)
    for (int i = tid; i < nown; i += bd) {
      const double x = __ldcg(r.T0 + n0 + i);
      sT[i] = x;
      st_stamped(r.ll[0] + 2 * (size_t)(n0 + i), x, r.stamp0);
    }
  }
  for (int64_t j = 0; j < r.nsteps; ++j) {
    const double *Tc = (j & 1) ? r.T1 : r.T0;
    double *Tn = (j & 1) ? r.T0 : r.T1;
    const unsigned long long step_no = (unsigned long long)(r.step0 + j + 1);
    const double t = j == 0 ? r.time0 : (double)(r.step0 + j) * r.dt;
    // 1. temperatures (and k(T), single material) of the owned + halo nodes;
    //    written by other CTAs in the previous step: L2 loads (no stale L1)
    if (STAMPED) {
      // the owned nodes are in sT already (the previous step's update); the
      // halo nodes arrive as stamped words from their owners.  A slot of
      // buffer j & 1 is rewritten by its owner in step j + 1, which the owner
      // starts only after every reader's step-j output (stamped after its reads) arrived.
      const unsigned long long *src = r.ll[j & 1];
      const uint32_t stamp = r.stamp0 + (uint32_t)j;
      for (int i = tid; i < nloc; i += bd) {
        double x;
        if (i < nown) {
          x = sT[i];
        } else if (!ld_stamped(src + 2 * (size_t)sH[i - nown], stamp, x, r.bar)) {
          s_bad = 2;  // lost a neighbour: this CTA leaves after the staging barrier
          x = 0.0;
        }
        if (i >= nown) sT[i] = x;
        if (TD && KSTAGE) sK[i] = interp_rn(k0, x);
      }
    } else {
      for (int i = tid; i < nloc; i += bd) {
        const int gi = i < nown ? n0 + i : sH[i - nown];
        FH_DEV_CHECK(gi >= 0 && gi < g.V, "resident staged node");
        const double x = __ldcg(Tc + gi);
        sT[i] = x;
        if (TD && KSTAGE) sK[i] = interp_rn(k0, x);
      }
    }
    __syncthreads();
    if (STAMPED && s_bad == 2) return;
    // 2. one contribution per incidence (k_exact_elem's arithmetic): the
    //    corner loads, differences and products are independent, only the
    //    sum runs in the reference's b order
    for (int q = tid; q < nq; q += bd) {
      const uint8_t info = sI[q];
      const uint4 w = reinterpret_cast<const uint4 *>(sL)[q];
      const int L[8] = {(int)(w.x & 0xffff), (int)(w.x >> 16), (int)(w.y & 0xffff), (int)(w.y >> 16),
                        (int)(w.z & 0xffff), (int)(w.z >> 16), (int)(w.w & 0xffff), (int)(w.w >> 16)};
      const double2 *A2 = reinterpret_cast<const double2 *>(sA + 8 * q);
#ifdef FH_CHECKS
      for (int b = 0; b < ((info & 8) ? 8 : 4); ++b) FH_DEV_CHECK(L[b] < nloc, "resident corner outside the staged nodes");
#endif
      if (info & 8) {
        double Tb[8], A[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) Tb[b] = sT[L[b]];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const double2 v = A2[b];
          A[2 * b] = v.x;
          A[2 * b + 1] = v.y;
        }
        double ke;
        if (TD) {
          const int e = sE[q];
          double s = 0.0;
          if (KSTAGE) {
#pragma unroll
            for (int b = 0; b < 8; ++b) s = add(s, sK[L[b]]);
          } else {
            const Curve<double> &kc = g.mats.m[g.elem_region ? g.elem_region[e] : 0].k;
#pragma unroll
            for (int b = 0; b < 8; ++b) s = add(s, interp_rn(kc, Tb[b]));
          }
          ke = dvd(s, 8.0);
          if (g.kfactor) ke = mul(ke, g.kfactor[e]);
        } else {
          ke = sKb[q];
        }
        double p[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) p[b] = mul(A[b], sub(Tb[b], Tb[0]));
        double acc = 0.0;
#pragma unroll
        for (int b = 0; b < 8; ++b) acc = add(acc, p[b]);
        sC[q] = mul(ke, acc);
      } else {
        double Tb[4], A[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) Tb[b] = sT[L[b]];
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const double2 v = A2[b];
          A[2 * b] = v.x;
          A[2 * b + 1] = v.y;
        }
        double ke;
        if (TD) {
          const int e = sE[q];
          double s = 0.0;
          if (KSTAGE) {
#pragma unroll
            for (int b = 0; b < 4; ++b) s = add(s, sK[L[b]]);
          } else {
            const Curve<double> &kc = g.mats.m[g.elem_region ? g.elem_region[e] : 0].k;
#pragma unroll
            for (int b = 0; b < 4; ++b) s = add(s, interp_rn(kc, Tb[b]));
          }
          ke = dvd(s, 4.0);
          if (g.kfactor) ke = mul(ke, g.kfactor[e]);
        } else {
          ke = sKb[q];
        }
        double p[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) p[b] = mul(A[b], sub(Tb[b], Tb[0]));
        double acc = 0.0;
#pragma unroll
        for (int b = 0; b < 4; ++b) acc = add(acc, p[b]);
        sC[q] = mul(ke, acc);
      }
    }
    __syncthreads();
    // 3. chunked sum per owned node (k_exact_node's order), update, runaway
    bool bad = false;
    for (int i = tid; i < nown; i += bd) {
      const int qs = sO[i], qe = sO[i + 1];
      // bit 4 of the info byte: this incidence opens a new 4096-element chunk
      // of the node's list (precomputed: no division per step)
      double total = 0.0, part = 0.0;
      for (int q = qs; q < qe; ++q) {
        if (sI[q] & 16) {
          if (q > qs) total = add(total, part);
          part = 0.0;
        }
        part = sub(part, sC[q]);
      }
      if (qe > qs) total = add(total, part);
      const int gi = n0 + i;
      if (g.F) g.F[gi] = total;
      const double xn = exact_update_in(g, sN[i], total, sT[i], r.dt, t, TD ? 1 : 0);
      if (STAMPED) st_stamped(r.ll[(j + 1) & 1] + 2 * (size_t)gi, xn, r.stamp0 + (uint32_t)j + 1u);
      else Tn[gi] = xn;
      sT[i] = xn;  // the next step and the probes below read the owned nodes' new values
      bad |= !isfinite(xn) || fabs(xn) > g.runaway_limit;
    }
    if (__any_sync(0xffffffffu, bad) && (tid & 31) == 0) {
      atomicMin(&g.flag->step, step_no);
      if (!STAMPED) s_bad = 1;
    }
    // probe record of this step, written by the CTA owning each probe node
    // (k_gather_probes' values; a failing step's record is dropped by the host)
    if (r.n_probes && step_no % (unsigned long long)r.probe_interval == 0) {
      const int64_t rec = r.rec0 + (int64_t)(step_no / r.probe_interval) -
                          (int64_t)((unsigned long long)r.step0 / r.probe_interval) - 1;
      if (rec < r.rec_cap) {
        __syncthreads();  // sT of the owned nodes holds the new field
        for (int64_t p = tid; p < r.n_probes; p += bd) {
          const int loc = r.probes[p] - n0;
          if (loc >= 0 && loc < nown) r.probe_out[rec * r.n_probes + p] = sT[loc];
        }
      }
    }
    if (STAMPED) {
      // no barrier: sT's owned entries are next read after the staging barrier
      // of the next step, its halo entries and sK only rewritten before it
      continue;
    }
    if (grid_barrier(r.bar, (unsigned long long)(j + 1) * gridDim.x, s_bad != 0, &s_word)) {
      done = j + 1;  // this step failed somewhere: its field is complete, stop here
      break;
    }
  }
  if (STAMPED) {
    // the engine's field: every CTA's owned nodes after the last step
    __syncthreads();
    for (int i = tid; i < nown; i += bd) r.T0[n0 + i] = sT[i];
    return;
  }
  // the field after the last completed step is in T1 when that count is odd
  if (done & 1)
    for (int i = tid; i < nown; i += bd) r.T0[n0 + i] = __ldcg(r.T1 + n0 + i);
}

template <bool TD, bool KSTAGE, bool STAMPED>
static void launch_one(const ResidentArgs &r, int n_cta, int threads, size_t smem, cudaStream_t s) {
  auto kern = k_resident<TD, KSTAGE, STAMPED>;
  static size_t configured = 0;
  if (smem > configured) {
    FH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = smem;
  }
  void *args[] = {const_cast<ResidentArgs *>(&r)};
  FH_CUDA(cudaLaunchCooperativeKernel((const void *)kern, dim3(n_cta), dim3(threads), args, smem, s));
}

void resident_run(const ResidentArgs &r, int n_cta, int threads, size_t smem, bool td, bool stage_k,
                  cudaStream_t s) {
  if (r.nsteps <= 0) return;
  if (r.ll[0]) {
    if (td && stage_k) launch_one<true, true, true>(r, n_cta, threads, smem, s);
    else if (td) launch_one<true, false, true>(r, n_cta, threads, smem, s);
    else launch_one<false, false, true>(r, n_cta, threads, smem, s);
    return;
  }
  if (td && stage_k) launch_one<true, true, false>(r, n_cta, threads, smem, s);
  else if (td) launch_one<true, false, false>(r, n_cta, threads, smem, s);
  else launch_one<false, false, false>(r, n_cta, threads, smem, s);
}

template <bool TD, bool KSTAGE>
static int occ_one(int threads, size_t smem) {
  // both synchronisation variants of a (TD, KSTAGE) pair: the smaller count decides
  auto kern2 = k_resident<TD, KSTAGE, true>;
  FH_CUDA(cudaFuncSetAttribute(kern2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int bps2 = 0;
  FH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps2, kern2, threads, smem));
  auto kern = k_resident<TD, KSTAGE, false>;
  FH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int bps = 0;
  FH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, threads, smem));
  return std::min(bps, bps2);
}

int resident_occupancy(bool td, bool stage_k, int threads, size_t smem) {
  if (td && stage_k) return occ_one<true, true>(threads, smem);
  if (td) return occ_one<true, false>(threads, smem);
  return occ_one<false, false>(threads, smem);
}

// ---------------------------------------------------------------------------
static size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

bool build_resident_plan(int64_t V, int64_t n_tet, int64_t chunk_size, const std::vector<int32_t> &conn,
                         const std::vector<int32_t> &csr_offs, const std::vector<int32_t> &csr_pos, int n_cta,
                         bool stage_k, bool frozen_kbar_slots, size_t smem_limit, ResidentPlan &P) {
  P = ResidentPlan{};
  const int64_t n_inc = csr_offs[V];
  n_cta = (int)std::max<int64_t>(1, std::min<int64_t>(n_cta, V));
  // contiguous node ranges with about n_inc / n_cta incidences each
  P.cta_node.assign(1, 0);
  for (int c = 1; c < n_cta; ++c) {
    const int64_t target = n_inc * c / n_cta;
    int64_t lo = P.cta_node.back() + 1, hi = V - (n_cta - c);
    if (lo > hi) return false;
    int64_t i = std::lower_bound(csr_offs.begin() + lo, csr_offs.begin() + hi + 1, (int32_t)target) - csr_offs.begin();
    P.cta_node.push_back((int32_t)std::min(std::max(i, lo), hi));
  }
  P.cta_node.push_back((int32_t)V);
  P.n_cta = n_cta;
  auto elem_of = [&](int64_t p) { return p < 4 * n_tet ? p / 4 : n_tet + (p - 4 * n_tet) / 8; };
  auto eoff = [&](int64_t e) { return e < n_tet ? 4 * e : 4 * n_tet + 8 * (e - n_tet); };
  P.cta_halo.assign(1, 0);
  P.cta_inc.assign(1, 0);
  P.inc_lconn.assign(8 * (size_t)n_inc, 0);
  P.inc_elem.resize(n_inc);
  P.inc_info.resize(n_inc);
  std::vector<int32_t> local(V, -1), halo;
  for (int c = 0; c < n_cta; ++c) {
    const int32_t n0 = P.cta_node[c], n1 = P.cta_node[c + 1];
    for (int32_t i = n0; i < n1; ++i) local[i] = i - n0;
    halo.clear();
    for (int32_t q = csr_offs[n0]; q < csr_offs[n1]; ++q) {
      const int64_t p = csr_pos[q], e = elem_of(p), p0 = eoff(e);
      const int n = e < n_tet ? 4 : 8;
      for (int b = 0; b < n; ++b) {
        const int32_t v = conn[p0 + b];
        if (v < n0 || v >= n1) halo.push_back(v);
      }
    }
    std::sort(halo.begin(), halo.end());
    halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
    const int32_t nown = n1 - n0;
    for (size_t k = 0; k < halo.size(); ++k) local[halo[k]] = nown + (int32_t)k;
    if (nown + (int64_t)halo.size() > 65535) return false;
    for (int32_t q = csr_offs[n0]; q < csr_offs[n1]; ++q) {
      const int64_t p = csr_pos[q], e = elem_of(p), p0 = eoff(e);
      const int n = e < n_tet ? 4 : 8;
      for (int b = 0; b < n; ++b) P.inc_lconn[8 * (size_t)q + b] = (uint16_t)local[conn[p0 + b]];
      P.inc_elem[q] = (int32_t)e;
      P.inc_info[q] = (uint8_t)((p - p0) | (n == 8 ? 8 : 0));
    }
    for (int32_t i = n0; i < n1; ++i)  // chunk openings along each node's list (k_exact_node's chunk switch)
      for (int32_t q = csr_offs[i]; q < csr_offs[i + 1]; ++q) {
        const int64_t ch = P.inc_elem[q] / chunk_size;
        if (q == csr_offs[i] || ch != P.inc_elem[q - 1] / chunk_size) P.inc_info[q] |= 16;
    }
    P.halo_nodes.insert(P.halo_nodes.end(), halo.begin(), halo.end());
    P.cta_halo.push_back((int32_t)P.halo_nodes.size());
    P.cta_inc.push_back(csr_offs[n1]);
    P.max_local = std::max<int>(P.max_local, nown + (int)halo.size());
    P.max_own = std::max<int>(P.max_own, nown);
    P.max_inc = std::max<int>(P.max_inc, csr_offs[n1] - csr_offs[n0]);
    for (int32_t i = n0; i < n1; ++i) local[i] = -1;
    for (int32_t v : halo) local[v] = -1;
  }
  const size_t L = (size_t)P.max_local, Q = (size_t)P.max_inc;
  size_t off = align16(8 * L);
  P.off_K = off;
  if (stage_k) off = align16(off + 8 * L);
  P.off_A = off;
  off = align16(off + 64 * Q);
  P.off_C = off;
  off = align16(off + 8 * Q);
  P.off_Kb = off;
  if (frozen_kbar_slots) off = align16(off + 8 * Q);
  P.off_H = off;
  off = align16(off + 4 * L);
  P.off_N = off;
  off = align16(off + sizeof(NodeIn) * (size_t)P.max_own);
  P.off_O = off;
  off = align16(off + 4 * ((size_t)P.max_own + 1));
  P.off_L = off;
  off = align16(off + 16 * Q);
  P.off_E = off;
  off = align16(off + 4 * Q);
  P.off_I = off;
  off = align16(off + Q);
  P.smem = off;
  P.threads = (int)std::min<size_t>(kResThreads, std::max<size_t>(64, (std::max(Q, L) + 31) / 32 * 32));
  return P.smem <= smem_limit;
}

}  // namespace fh
