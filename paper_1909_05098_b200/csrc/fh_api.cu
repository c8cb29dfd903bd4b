#include <cstdarg>
// C ABI of libfedheat_b200.so (include/fedheat_b200.h): engine lifetime,
// device precompute, state I/O, stepping, probes, critical dt, operator layer.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>
#include <type_traits>

#include "fh_dist.h"
#include "fh_tiled.cuh"
#include "fh_resident.h"
#include <limits>
#include "fh_atomic.h"

using namespace fh;

namespace {

thread_local std::string g_last_error;

}  // namespace

int fh::set_error(int code, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

namespace {

int report(const std::exception &ex) {
  if (const auto *fe = dynamic_cast<const Error *>(&ex)) {
    g_last_error = fe->what();
    return fe->code;
  }
  g_last_error = ex.what();
  return FH_ERR_DEVICE;
}

#define FH_API_BEGIN try {
#define FH_API_END                   \
  }                                  \
  catch (const std::exception &ex) { \
    return report(ex);               \
  }                                  \
  return FH_OK;

template <typename S>
void fill_curve(Curve<S> &c, const fh_curve &src, const char *what, bool optional = false) {
  std::memset(&c, 0, sizeof(c));
  if (src.n == 0 && optional) return;
  if (src.n < 1 || src.n > FH_MAX_KNOTS)
    fail(FH_ERR_CONFIG, std::string(what) + ": curve needs 1.." + std::to_string(FH_MAX_KNOTS) + " knots");
  c.n = src.n;
  for (int j = 0; j < src.n; ++j) {
    c.x[j] = (S)src.x[j];
    c.y[j] = (S)src.y[j];
    if (j + 1 < src.n) {
      if (!(src.x[j + 1] > src.x[j])) fail(FH_ERR_CONFIG, std::string(what) + ": knots must increase");
      c.slope[j] = (S)((src.y[j + 1] - src.y[j]) / (src.x[j + 1] - src.x[j]));
    }
  }
}

template <typename S>
void fill_mats(MatSet<S> &ms, const fh_options &o) {
  std::memset(&ms, 0, sizeof(ms));
  if (o.n_materials < 1 || o.n_materials > kMaxRegions || !o.materials)
    fail(FH_ERR_CONFIG, "need 1.." + std::to_string(kMaxRegions) + " materials");
  ms.n = o.n_materials;
  for (int r = 0; r < o.n_materials; ++r) {
    const fh_material &m = o.materials[r];
    Mat<S> &d = ms.m[r];
    fill_curve(d.rho, m.density, "density");
    fill_curve(d.c, m.specific_heat, "specific_heat");
    fill_curve(d.k, m.conductivity, "conductivity");
    fill_curve(d.wb, m.perfusion, "perfusion", true);
    d.td_perf = m.perfusion.n > 0;
    d.wbcb = (S)(m.perfusion_rate * m.blood_specific_heat);
    d.cb = (S)m.blood_specific_heat;
    d.Ta = (S)m.arterial_temperature;
    d.Qm = (S)m.metabolic_rate;
  }
}

__global__ void k_to_new(const double *__restrict__ src_old, const int64_t *__restrict__ old_of_new, int64_t V,
                         float *__restrict__ df, double *__restrict__ dd, float *__restrict__ df2,
                         double *__restrict__ dd2) {
  const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (n >= V) return;
  const double v = src_old[old_of_new ? old_of_new[n] : n];
  if (df) df[n] = (float)v;
  if (dd) dd[n] = v;
  if (df2) df2[n] = (float)v;
  if (dd2) dd2[n] = v;
}

// TILED: Dirichlet values written into a temperature buffer (new numbering);
// the step kernel never updates these nodes, so they keep the values exactly
template <typename S>
__global__ void k_scatter_dir(S *T, const int32_t *__restrict__ ids, const S *__restrict__ vals, int64_t n) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q < n) T[ids[q]] = vals[q];
}

// a Dirichlet value beyond the runaway limit fails every step (the reference
// checks max |T| over all nodes after the overwrite, solver.py:369-370)
__global__ void k_flag_step(FailFlag *flag, unsigned long long step_no) { atomicMin(&flag->step, step_no); }

template <typename S>
__global__ void k_to_old(const S *__restrict__ src_new, const int64_t *__restrict__ new_of_old, int64_t V,
                         double *__restrict__ dst_old) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= V) return;
  const int64_t n = new_of_old ? new_of_old[i] : i;
  dst_old[i] = n >= 0 ? (double)src_new[n] : __longlong_as_double(0x7ff8000000000000ll);  // not in this rank's view
}

template <typename S>
__global__ void k_xyzv_to_new(const double *__restrict__ xyz, const int64_t *__restrict__ old_of_new,
                              const S *__restrict__ vol_new, int64_t V, S *__restrict__ out) {
  // packed (x, y, z, v) per node, new numbering: one vector load in the step kernel
  const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (n >= V) return;
  const int64_t o = old_of_new[n];
  out[4 * n] = (S)xyz[3 * o];
  out[4 * n + 1] = (S)xyz[3 * o + 1];
  out[4 * n + 2] = (S)xyz[3 * o + 2];
  out[4 * n + 3] = vol_new[n];
}

template <typename S>
__global__ void k_pack_slots(const int32_t *__restrict__ slot_elem, int64_t n, const double *__restrict__ G,
                             double scale, S *__restrict__ out_G, int rec_elems, int g_off, const double *__restrict__ kf,
                             S *__restrict__ out_kf, const int32_t *__restrict__ region,
                             uint8_t *__restrict__ out_region, int paired) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int64_t e = slot_elem[s];
  // G rows of the batch record: record s / B, element offset g_off, [component][s % B]
  const int64_t base = (s / kBatch) * rec_elems + g_off + (s % kBatch);
  // temperature-dependent runs fold the conductivity factor into G (no kf
  // stream: out_kf == nullptr); frozen runs keep it for the freeze
  const double f = (kf && !out_kf && e >= 0) ? kf[e] : 1.0;
  // G components 00 01 02 11 12 22: [6][B] rows, or (LEAN records) 3 rows of
  // interleaved pairs (00,01) (02,11) (12,22)
  const int64_t pbase = (s / kBatch) * rec_elems + g_off + 2 * (s % kBatch);
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const S v = e >= 0 ? (S)(G[6 * e + k] * scale * f) : S(0);
    if (paired) out_G[pbase + (k >> 1) * 2 * kBatch + (k & 1)] = v;
    else out_G[base + k * kBatch] = v;
  }
  if (out_kf) out_kf[s] = e >= 0 ? (S)kf[e] : S(1);
  if (out_region) out_region[s] = e >= 0 ? (uint8_t)region[e] : 0;
}

// fp32 LEAN 1 records: the 16-bit node references become byte offsets (x 4;
// tets keep their accumulator row in bits 14-15), see k_tiled_step
__global__ void k_scale_conn(unsigned char *rec, int64_t n_batches, int rec_bytes, int words_per_batch, int tagged) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_batches * words_per_batch) return;
  uint16_t *w = reinterpret_cast<uint16_t *>(rec + (i / words_per_batch) * rec_bytes) + i % words_per_batch;
  const uint16_t v = *w;
  *w = tagged ? (uint16_t)((v & 0xc000u) | ((v & 0x3fffu) << 2)) : (uint16_t)(v << 2);
}

constexpr int kBlk = 256;
inline unsigned nblk(int64_t n) { return (unsigned)((n + kBlk - 1) / kBlk); }

template <typename S>
struct TiledState {
  TiledArgs<S> args{};
  DBuf<int32_t> part_node_start, part_n_free, part_robin_start, part_robin_base, part_tet_start, part_hex_start;
  DBuf<int32_t> part_tet_count, part_hex_count, part_halo_start, halo_nodes;
  DBuf<int32_t> part_list;
  DBuf<unsigned char> tet_rec, hex_rec;  // per-batch [conn16 | G] records (RecBytes)
  DBuf<int32_t> tet_conn, hex_conn, tet_slot_elem, hex_slot_elem;
  DBuf<S> tet_kf, hex_kf, tet_kbar, hex_kbar;
  DBuf<uint8_t> tet_rank, hex_rank, tet_region, hex_region, node_region;
  DBuf<int8_t> part_mat, part_region;
  DBuf<uint8_t> tet_phase, hex_phase, tet_bnph, hex_bnph;
  DBuf<S> T[2], vol, cap, kb, q_ext, xyz, robin_hA, robin_hAT;
  DBuf<int32_t> dir_ids;  // Dirichlet nodes (new numbering) and their values
  DBuf<S> dir_vals, F;    // F: net conduction inflow of the updated nodes (ExplicitEngine.step)
  bool dir_pending = false;  // T[cur] (the field as set) still lacks the Dirichlet values
  int cur = 0;
  size_t smem = 0;
  int n_parts_local = 0;
  int n_boundary = 0;  // multi-GPU: leading entries of part_list that touch the halo
  // tiles with tets at the head of the boundary / interior ranges (mixed meshes)
  int n_mixed_b = 0, n_mixed_i = 0;
  int n_lean_i = 0;  // one GPU, regions / mixed mesh: material-0 hex-only tiles at the end of the list (LEAN 2 launch)
  int n_lean_mixed_i = 0;  // ... and the material-0 tiles holding tets, at the end of the mixed range (LEAN 3 launch)
  int mode = 0;
  bool lean = false;  // LEAN loops and their paired-G records
};

}  // namespace

struct fh_engine {
  int device = 0;
  cudaStream_t stream = nullptr;
  int precision = 64, assembly = FH_ASSEMBLY_EXACT;
  bool td = false;
  int64_t V = 0, E = 0, n_tet = 0, n_hex = 0, nconn = 0;
  int64_t Vt = 0;  // TILED: nodes of the device node arrays (V, or the rank's owned + halo nodes)
  double runaway_limit = 1e6;
  bool dir_runaway = false;  // some |Dirichlet value| > runaway_limit: every step fails
  bool keep_inflow = false;  // TILED: the step kernel also writes F (fh_keep_inflow)
  bool io_failed = false;    // an async step failed: fh_set_temperature must come first
  double io_dt = 0.0;        // dt of the last fh_step_host_async (clock rollback on failure)
  int64_t step_index = 0;
  double time = 0.0;
  bool frozen = false;
  fh_options opts{};
  MatSet<double> mats_d{};
  MatSet<float> mats_f{};
  // boundary (host)
  std::vector<int64_t> dir_nodes;
  std::vector<double> dir_vals;
  std::vector<int64_t> load_offs, load_nodes;
  std::vector<double> load_power, load_t0, load_t1;
  std::vector<uint8_t> load_sig;
  bool qr_valid = false;
  std::vector<double> q_static;
  std::vector<fh_source> sources;
  std::vector<int64_t> robin_nodes;
  std::vector<double> robin_hA, robin_hAT;
  std::vector<double> host_xyz;
  // common device data (original numbering)
  DBuf<double> xyz, node_vol, elem_vol, row_abs, stage, stage2;
  DBuf<int32_t> conn, csr_offs, csr_pos, elem_region, node_region;
  DBuf<double> kfactor;
  DBuf<FailFlag> flag;
  // exact
  ExactArgs ex{};
  DBuf<double> A, kbar, cap, kb, qb, qm, qr, qstat, contrib, F, T, dir_vals_d, robin_hA_d, robin_hAT_d;
  DBuf<int32_t> dir_slot, robin_slot;
  // resident small-mesh EXACT path (fh_resident.cu)
  bool resident = false, res_stage_k = false;
  int res_ctas = 0, res_threads = 0;
  size_t res_smem = 0;
  ResidentArgs res{};
  DBuf<int32_t> r_cta_node, r_cta_halo, r_halo, r_cta_inc, r_inc_elem;
  DBuf<uint16_t> r_lconn;
  DBuf<uint8_t> r_info;
  DBuf<double> T1;
  DBuf<unsigned long long> r_bar;
  DBuf<unsigned long long> r_ll[2];  // stamped-word buffers of the resident kernel (2 words per node)
  uint32_t r_epoch = 1;              // next unused stamp (0 = never written)
  DBuf<double> r_snap;               // field at the start of a call (replay after a runaway)
  // ATOMIC assembly (fh_atomic.cu): element streams in the TILED numbering
  AtomicState atom;
  DBuf<int32_t> a_tet_conn, a_hex_conn;
  DBuf<char> a_tet_G, a_hex_G, a_F, a_hA, a_hAT;
  DBuf<uint8_t> a_cls;
  // tiled
  Partition part;
  DBuf<int64_t> old_of_new, new_of_old;
  std::unique_ptr<TiledState<float>> tf;
  std::unique_ptr<TiledState<double>> tdd;
  // multi-GPU halo exchange (fh_dist.cu)
  Exchange X;
  DBuf<int32_t> x_send, x_recv;
  DBuf<char> x_sendbuf, x_recvbuf;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_packed = nullptr, ev_halo = nullptr;
  bool halo_pending = false;
  void *comm = nullptr;  // ncclComm_t
  fh_transport transport{};  // host transport (fh_attach_transport), instead of NCCL
  DBuf<unsigned long long> red_scratch;  // NCCL all-reduce of host values
  std::vector<char> x_host_send, x_host_recv;
  DBuf<char> snap;  // multi-GPU: the field at the start of an fh_step call (exact failure replay)
  // probes
  DBuf<int32_t> probes;
  int64_t n_probes = 0, probe_interval = 1, probe_cap = 0, n_rec = 0;
  DBuf<double> probe_hist;
  std::vector<int64_t> probe_steps;
  // critical dt scratch
  DBuf<double> crit_kbar, crit_lam;
  // double-buffered host I/O (fh_step_host_async / fh_host_wait): per slot an
  // input and an output staging field, copy streams in each direction
  DBuf<double> io_in[2], io_out[2];
  cudaStream_t io_h2d = nullptr, io_d2h = nullptr;
  cudaEvent_t io_ev[2][4] = {};  // in ready, in consumed, out ready, out copied
  bool io_used[2] = {false, false};
  FailFlag *io_flag = nullptr;  // pinned: the fail flag after each slot's steps
  int refit_per_sm = 0;          // wave fit: measured resident step CTAs per SM (second pass)
  cudaStream_t kind_stream = nullptr;  // mixed meshes: the mixed-tile launch runs beside the hex-only one
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;

  ~fh_engine() {
    if (io_flag) cudaFreeHost(io_flag);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (kind_stream) cudaStreamDestroy(kind_stream);
    for (auto &evs : io_ev)
      for (cudaEvent_t ev : evs)
        if (ev) cudaEventDestroy(ev);
    if (io_h2d) cudaStreamDestroy(io_h2d);
    if (io_d2h) cudaStreamDestroy(io_d2h);
    if (comm) nccl_comm_destroy(comm);
    if (ev_packed) cudaEventDestroy(ev_packed);
    if (ev_halo) cudaEventDestroy(ev_halo);
    if (comm_stream) cudaStreamDestroy(comm_stream);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

void check_engine(fh_engine *e) {
  if (!e) fail(FH_ERR_CONFIG, "null engine");
  FH_CUDA(cudaSetDevice(e->device));
}

// q_r from the active heat loads (solver.py:307-318) + static nodal power
bool loads_changed(fh_engine *e, double t) {
  const int64_t nl = (int64_t)e->load_power.size();
  bool changed = !e->qr_valid;
  for (int64_t l = 0; l < nl; ++l) {
    const uint8_t on = (e->load_t0[l] <= t && t < e->load_t1[l]);
    if (on != e->load_sig[l]) changed = true;
    e->load_sig[l] = on;
  }
  e->qr_valid = true;
  return changed;
}

std::vector<double> dense_qr(fh_engine *e) {
  std::vector<double> qr(e->V, 0.0);
  for (size_t l = 0; l < e->load_power.size(); ++l)
    if (e->load_sig[l])
      for (int64_t q = e->load_offs[l]; q < e->load_offs[l + 1]; ++q) qr[e->load_nodes[q]] += e->load_power[l];
  return qr;
}

template <typename S>
TiledState<S> &tstate(fh_engine *e);
template <>
TiledState<float> &tstate<float>(fh_engine *e) { return *e->tf; }
template <>
TiledState<double> &tstate<double>(fh_engine *e) { return *e->tdd; }

// Default tile size (nodes per part), from scripts/sweep.py on B200: fp32 hex
// meshes 1536 (cfg4, cfg5), tet meshes 768 (~6 tets per node: the same slots
// per tile at half the nodes; cfg3), fp64 768.
int default_part_nodes(int precision, int64_t n_tet, int64_t n_hex) {
  if (precision != 32) return 768;
  return n_tet > n_hex ? 768 : 1536;
}

// Tet-only meshes: colour classes with up to 4 writes per node (4 accumulator
// rows, ~4x larger classes -> fewer colour phases per 256-slot batch).  fp64
// keeps 3 rows: the row saved lets a fourth tile CTA fit each SM's shared
// memory (cfg3 fp64 0.1068 -> 0.1000 ms/step; 2 rows 0.1008).
int default_tet_rows(int64_t n_tet, int64_t n_hex, int knob, int precision) {
  int r = (n_tet > 0 && n_hex == 0) ? (precision == 32 ? 4 : 3) : 1;
  if (knob > 0) r = std::min(knob, 4);  // fh_options.tet_rows
  return r;
}

// Wave fit: with only a few waves of tile CTAs per launch, the last partial
// wave leaves SMs idle (cfg3: 1342 tiles on 148 SMs x 5 CTAs = 1.81 waves).
// The tile size is lowered just enough that the tile count fills the last wave
// (cfg3: 1480 tiles, 0.0923 -> 0.089 ms/step; scripts/sweep.py).  Parts per
// domain are ceil(V_domain / target) (fh_partition.cpp), so the count is exact.
int wave_fit_part_nodes(int target, int64_t V, int n_domains, int precision, int64_t n_tet, int64_t n_hex,
                        int device, int per_sm_measured = 0) {
  int sms = 148;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || sms <= 0) {
    cudaGetLastError();
    sms = 148;
  }
  // resident step CTAs per SM (the launch bounds of k_tiled_step)
  // (the launch bounds' minimum; setup_tiled refits with the measured value)
  const int per_sm = per_sm_measured > 0 ? per_sm_measured : (precision != 32 ? 2 : (n_hex == 0 ? 6 : 5));
  const int64_t cap = (int64_t)sms * per_sm;
  const int64_t vd = (V + n_domains - 1) / n_domains;
  const int64_t n0 = (int64_t)n_domains * ((vd + target - 1) / target);
  const double waves = (double)n0 / (double)cap;
  if (waves >= 6.0) return target;  // the tail is a small fraction already
  const int64_t w = (int64_t)std::ceil(waves - 1e-9);
  const int64_t per_dom = std::max<int64_t>(1, w * cap / n_domains);
  const int64_t t = (vd + per_dom - 1) / per_dom;
  return (int)std::max<int64_t>(64, std::min<int64_t>(target, t));
}

// Tiled kernels: a one-knot curve becomes the two-knot curve (y0, y0) with
// slope 0 (same values everywhere).  Returns 1 when every curve of every
// material then has exactly two knots (branch-free interpolation kernels).
template <typename S>
int normalise_curves(MatSet<S> &ms) {
  int lin = 1;
  for (int r = 0; r < ms.n; ++r) {
    Curve<S> *cs[4] = {&ms.m[r].rho, &ms.m[r].c, &ms.m[r].k, &ms.m[r].wb};
    for (Curve<S> *c : cs) {
      if (c->n == 0) continue;  // no perfusion law (constant perfusion)
      if (c->n == 1) {
        c->n = 2;
        c->x[1] = c->x[0];
        c->y[1] = c->y[0];
        c->slope[0] = S(0);
      }
      if (c->n != 2) lin = 0;
    }
  }
  return lin;
}

template <typename S>
MatSet<S> &mats_of(fh_engine *e);
template <>
MatSet<float> &mats_of<float>(fh_engine *e) { return e->mats_f; }
template <>
MatSet<double> &mats_of<double>(fh_engine *e) { return e->mats_d; }

void upload_qr(fh_engine *e, double t) {
  if (e->load_power.empty()) return;
  if (!loads_changed(e, t)) return;
  std::vector<double> qr = dense_qr(e);
  FH_CUDA(cudaStreamSynchronize(e->stream));
  if (e->assembly == FH_ASSEMBLY_EXACT) {
    FH_CUDA(cudaMemcpy(e->qr.p, qr.data(), sizeof(double) * e->V, cudaMemcpyHostToDevice));
    return;
  }
  if (!e->q_static.empty())
    for (int64_t i = 0; i < e->V; ++i) qr[i] += e->q_static[i];
  FH_CUDA(cudaMemcpy(e->stage.p, qr.data(), sizeof(double) * e->V, cudaMemcpyHostToDevice));
  if (e->precision == 32)
    k_to_new<<<nblk(e->Vt), kBlk>>>(e->stage.p, e->old_of_new.p, e->Vt, e->tf->q_ext.p, nullptr, nullptr, nullptr);
  else
    k_to_new<<<nblk(e->Vt), kBlk>>>(e->stage.p, e->old_of_new.p, e->Vt, nullptr, e->tdd->q_ext.p, nullptr, nullptr);
  FH_CUDA(cudaGetLastError());
  FH_CUDA(cudaDeviceSynchronize());
}

// ---------------------------------------------------------------------------
void setup_exact(fh_engine *e, const fh_boundary &b) {
  cudaStream_t s = e->stream;
  const int64_t V = e->V;
  ExactArgs &g = e->ex;
  std::memset(&g, 0, sizeof(g));
  g.V = V;
  g.E = e->E;
  g.n_tet = e->n_tet;
  g.chunk_size = FH_CHUNK_SIZE;
  g.conn = e->conn.p;
  g.mat = e->A.p;
  g.row_abs = e->row_abs.p;
  g.csr_offs = e->csr_offs.p;
  g.csr_pos = e->csr_pos.p;
  g.node_vol = e->node_vol.p;
  g.elem_region = e->elem_region.p;
  g.node_region = e->node_region.p;
  g.kfactor = e->kfactor.p;
  g.mats = e->mats_d;
  e->kbar.alloc(e->E);
  e->cap.alloc(V);
  e->contrib.alloc(e->nconn);
  e->F.alloc(V);
  e->F.zero(s);
  e->T.alloc(V);
  e->qr.alloc(V);
  e->qr.zero(s);
  g.kbar = e->kbar.p;
  g.cap = e->cap.p;
  g.contrib = e->contrib.p;
  g.F = e->F.p;
  g.qr = e->qr.p;
  // constant lumps (precompute.py:43-53): kb = (wb*cb)*v, qb = kb*Ta, qm = Qm*v
  std::vector<double> nv(V), kbh(V), qbh(V), qmh(V);
  FH_CUDA(cudaMemcpyAsync(nv.data(), e->node_vol.p, sizeof(double) * V, cudaMemcpyDeviceToHost, s));
  std::vector<int32_t> nreg(V, 0);
  if (e->node_region.p)
    FH_CUDA(cudaMemcpyAsync(nreg.data(), e->node_region.p, sizeof(int32_t) * V, cudaMemcpyDeviceToHost, s));
  FH_CUDA(cudaStreamSynchronize(s));
  for (int64_t i = 0; i < V; ++i) {
    const fh_material &m = e->opts.materials[nreg[i]];
    kbh[i] = (m.perfusion_rate * m.blood_specific_heat) * nv[i];
    qbh[i] = kbh[i] * m.arterial_temperature;
    qmh[i] = m.metabolic_rate * nv[i];
  }
  e->kb.upload(kbh, s);
  e->qb.upload(qbh, s);
  e->qm.upload(qmh, s);
  g.kb = e->kb.p;
  g.qb = e->qb.p;
  g.qm = e->qm.p;
  if (!e->q_static.empty()) {
    e->qstat.upload(e->q_static, s);
    g.q_static = e->qstat.p;
  }
  std::vector<int32_t> ds(V, -1);
  for (size_t q = 0; q < e->dir_nodes.size(); ++q) ds[e->dir_nodes[q]] = (int32_t)q;
  if (!e->dir_nodes.empty()) {
    e->dir_slot.upload(ds, s);
    e->dir_vals_d.upload(e->dir_vals, s);
    g.dir_slot = e->dir_slot.p;
    g.dir_vals = e->dir_vals_d.p;
  }
  if (!e->robin_nodes.empty()) {
    std::vector<int32_t> rs(V, -1);
    for (size_t q = 0; q < e->robin_nodes.size(); ++q) rs[e->robin_nodes[q]] = (int32_t)q;
    e->robin_slot.upload(rs, s);
    e->robin_hA_d.upload(e->robin_hA, s);
    e->robin_hAT_d.upload(e->robin_hAT, s);
    g.robin_slot = e->robin_slot.p;
    g.robin_hA = e->robin_hA_d.p;
    g.robin_hAT = e->robin_hAT_d.p;
  }
  g.xyz = e->xyz.p;
  g.n_src = (int)e->sources.size();
  for (int k = 0; k < g.n_src; ++k) g.src[k] = e->sources[k];
  g.runaway_limit = e->runaway_limit;
  g.flag = e->flag.p;
  FH_CUDA(cudaStreamSynchronize(s));
}

// The resident path (fh_resident.cu) when every CTA's working set fits
// shared memory and the grid stays co-resident (one CTA per SM by default).
void setup_resident(fh_engine *e, const std::vector<int32_t> &conn, const std::vector<int32_t> &offs,
                    const std::vector<int32_t> &pos) {
  const fh_options &o = e->opts;
  if (o.resident_sync < 0 || o.resident_sync > 1) fail(FH_ERR_CONFIG, "resident_sync must be 0 or 1");
  if (o.exact_resident == 1) return;
  int sms = 148, smem_optin = 227 * 1024;
  FH_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, e->device));
  FH_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, e->device));
  const bool stage_k = e->td && !(o.n_materials > 1 && o.element_region);
  // CTA count: the knob, else two per SM with stamped halo words (measured:
  // cfg1 2.39 -> 2.25 us/step, cfg2 3.56 -> 3.21 over one per SM; the grid
  // barrier is fastest with one per SM), falling back to one per SM when two
  // do not stay co-resident
  std::vector<int> tries;
  if (o.resident_ctas > 0) tries = {o.resident_ctas};
  else if (o.resident_sync == 0) tries = {2 * sms, sms};
  else tries = {sms};
  ResidentPlan P;
  bool ok = false;
  for (int ctas : tries) {
    ok = build_resident_plan(e->V, e->n_tet, FH_CHUNK_SIZE, conn, offs, pos, ctas, stage_k, !e->td,
                             (size_t)smem_optin - 1024, P);
    if (ok) ok = (int64_t)resident_occupancy(e->td, stage_k, P.threads, P.smem) * sms >= P.n_cta;
    if (ok) break;
  }
  if (!ok) {
    if (o.exact_resident == 2) fail(FH_ERR_CONFIG, "the resident EXACT path does not fit this mesh");
    return;
  }
  cudaStream_t s = e->stream;
  e->r_cta_node.upload(P.cta_node, s);
  e->r_cta_halo.upload(P.cta_halo, s);
  e->r_halo.upload(P.halo_nodes.empty() ? std::vector<int32_t>{0} : P.halo_nodes, s);
  e->r_cta_inc.upload(P.cta_inc, s);
  e->r_inc_elem.upload(P.inc_elem, s);
  e->r_lconn.upload(P.inc_lconn, s);
  e->r_info.upload(P.inc_info, s);
  e->T1.alloc(e->V);
  e->r_bar.alloc(1);
  e->r_bar.zero(s);
  ResidentArgs &r = e->res;
  std::memset(&r, 0, sizeof(r));
  r.cta_node = e->r_cta_node.p;
  r.cta_halo = e->r_cta_halo.p;
  r.halo_nodes = e->r_halo.p;
  r.cta_inc = e->r_cta_inc.p;
  r.inc_lconn = e->r_lconn.p;
  r.inc_elem = e->r_inc_elem.p;
  r.inc_info = e->r_info.p;
  r.off_K = (uint32_t)P.off_K;
  r.off_A = (uint32_t)P.off_A;
  r.off_C = (uint32_t)P.off_C;
  r.off_Kb = (uint32_t)P.off_Kb;
  r.off_L = (uint32_t)P.off_L;
  r.off_E = (uint32_t)P.off_E;
  r.off_I = (uint32_t)P.off_I;
  r.off_H = (uint32_t)P.off_H;
  r.off_N = (uint32_t)P.off_N;
  r.off_O = (uint32_t)P.off_O;
  r.T0 = e->T.p;
  r.T1 = e->T1.p;
  r.bar = e->r_bar.p;
  if (o.resident_sync != 1) {  // stamped halo words instead of a grid barrier per step
    for (int q = 0; q < 2; ++q) {
      e->r_ll[q].alloc(2 * (size_t)e->V);
      e->r_ll[q].zero(s);
      r.ll[q] = e->r_ll[q].p;
    }
    e->r_snap.alloc(e->V);
  }
  e->resident = true;
  e->res_stage_k = stage_k;
  e->res_ctas = P.n_cta;
  e->res_threads = P.threads;
  e->res_smem = P.smem;
  FH_CUDA(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------------------
template <typename S>
void setup_tiled(fh_engine *e, const fh_mesh &mesh, const fh_boundary &b, const double *G_dev) {
  cudaStream_t s = e->stream;
  const int64_t V = e->V;
  const fh_options &o = e->opts;
  // node classes
  std::vector<uint8_t> cls(V, 0);
  for (int64_t i : e->robin_nodes) cls[i] = 1;
  for (int64_t i : e->dir_nodes) cls[i] = 2;
  PartitionInput pin{};
  pin.V = V;
  pin.n_tet = e->n_tet;
  pin.n_hex = e->n_hex;
  pin.xyz = mesh.coords;
  pin.tets = mesh.tets;
  pin.hexes = mesh.hexes;
  pin.node_class = cls.data();
  pin.target_part_nodes = o.part_nodes > 0 ? o.part_nodes : default_part_nodes(sizeof(S) == 4 ? 32 : 64, e->n_tet, e->n_hex);
  // small meshes: shrink the tiles so that at least ~2 CTAs per SM exist (latency-bound regime)
  if (o.part_nodes <= 0 && V / pin.target_part_nodes < 2 * 148)
    pin.target_part_nodes = (int)std::max<int64_t>(96, V / (2 * 148));
  else if (o.part_nodes <= 0)
    pin.target_part_nodes = wave_fit_part_nodes(pin.target_part_nodes, V, std::max(1, o.n_domains),
                                                sizeof(S) == 4 ? 32 : 64, e->n_tet, e->n_hex, o.device,
                                                e->refit_per_sm);
  const int target_used = pin.target_part_nodes;
  pin.batch = kBatch;
  // layout tuning knobs (fh_options; scripts/sweep.py): hex colour order, first-touch node order
  pin.hex_color = o.hex_color;
  pin.first_touch = o.first_touch;
  pin.tet_rows = default_tet_rows(e->n_tet, e->n_hex, o.tet_rows, sizeof(S) == 4 ? 32 : 64);
  pin.n_domains = std::max(1, o.n_domains);
  pin.slab_axis = o.slab_axis;
  build_partition(pin, e->part);
  Partition &P = e->part;

  auto st = std::make_unique<TiledState<S>>();
  TiledArgs<S> &g = st->args;
  std::memset(&g, 0, sizeof(g));
  // parts of this engine: domains [lo, hi) = rank `lo / width` of `D / width`
  const int D = pin.n_domains;
  const int dlo = std::max(0, o.domain_lo), dhi = o.domain_hi > 0 ? o.domain_hi : D;
  const int width = dhi - dlo;
  if (width < 1 || dhi > D || D % width != 0 || dlo % width != 0)
    fail(FH_ERR_CONFIG, "domain range must be one of D/width equal blocks");
  {
    std::vector<uint8_t> is_dir(e->V, 0);
    for (int64_t i : e->dir_nodes) is_dir[P.new_of_old[i]] = 1;
    build_exchange(P, is_dir.data(), D, D / width, dlo / width, e->X);
  }
  // multi-GPU: keep only this rank's parts, slots and the nodes they read
  // (local numbering: owned range, then the foreign halo nodes), so the
  // per-step device working set is the rank's share of the mesh
  if (e->X.world > 1) {
    Partition Lp;
    localize_partition(P, e->X, Lp);
    P = std::move(Lp);
  }
  const int64_t Vt = (int64_t)P.old_of_new.size();  // nodes of the tiled arrays (V on one GPU)
  e->Vt = Vt;
  e->old_of_new.upload(P.old_of_new, s);
  e->new_of_old.upload(P.new_of_old, s);
  std::vector<int32_t> plist = e->X.part_order;  // boundary tiles first
  st->n_parts_local = (int)plist.size();
  st->n_boundary = e->X.world > 1 ? e->X.n_boundary : 0;
  // launches of a few waves: longest tiles first inside each launch range
  // (CTAs are dispatched in order, so the short tiles fill the last wave;
  // cfg3 0.0865 -> 0.0843 ms/step).  Long launches keep the RCB order: there
  // the spatial order's L2 reuse of halo temperatures wins (cfg4 +7% slower).
  int sms = 148;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, o.device) != cudaSuccess) {
    cudaGetLastError();
    sms = 148;
  }
  const int per_sm = e->refit_per_sm > 0 ? e->refit_per_sm
                                         : (sizeof(S) == 4 ? (e->n_hex == 0 ? 6 : 5) : 2);
  bool lpt = (double)plist.size() / ((double)sms * per_sm) < 6.0;
  if (o.launch_order) lpt = o.launch_order == 2;
  if (lpt) {
    auto work = [&](int32_t p) { return (int64_t)P.part_tet_count[p] + 2 * (int64_t)P.part_hex_count[p]; };
    auto by_work = [&](int32_t a, int32_t b) { return work(a) > work(b); };
    std::stable_sort(plist.begin(), plist.begin() + st->n_boundary, by_work);
    std::stable_sort(plist.begin() + st->n_boundary, plist.end(), by_work);
  }
  // mixed meshes: inside each launch range the tiles holding tets come first,
  // so the hex-only tiles can run the leaner hex-only kernel instance
  const bool has_regions = o.n_materials > 1 && o.element_region;
  bool split = e->n_tet > 0 && e->n_hex > 0;
  // a hex-only mesh with material regions splits the same way on one GPU (no
  // tile holds tets), so that its region-0 tiles can run the LEAN 2 loop below
  if (e->n_tet == 0 && e->n_hex > 0 && has_regions && e->X.world == 1) split = true;
  if (o.kind_split == 1) split = false;
  st->n_mixed_b = st->n_boundary;
  st->n_mixed_i = st->n_parts_local - st->n_boundary;
  if (split) {
    auto has_tet = [&](int32_t p) { return P.part_tet_count[p] > 0; };
    auto mid_b = std::stable_partition(plist.begin(), plist.begin() + st->n_boundary, has_tet);
    auto mid_i = std::stable_partition(plist.begin() + st->n_boundary, plist.end(), has_tet);
    st->n_mixed_b = (int)(mid_b - plist.begin());
    st->n_mixed_i = (int)(mid_i - (plist.begin() + st->n_boundary));
  }
  // one GPU, a mesh with material regions or with both element kinds: the
  // hex-only tiles whose slots all lie in region 0 go last and run the LEAN 2
  // loop (fh_tiled.cu); the region-0 tiles that hold tets go to the end of the
  // mixed range and run the LEAN 3 loop; the others keep the general kernel
  if (e->X.world == 1 && (has_regions || split) && e->td && o.lean_kernels == 0 && o.tile_mode == 0 &&
      P.corner_unique && sizeof(S) == 4 && !(e->kfactor.p && !e->td)) {
    MatSet<S> mt = mats_of<S>(e);
    bool ok = normalise_curves(mt) != 0;
    for (int q = 0; q < P.n_parts && ok; ++q)
      ok = (P.part_hex_count[q] + kBatch - 1) / kBatch + (P.part_tet_count[q] + kBatch - 1) / kBatch <= kBatch;
    auto region0 = [&](int32_t p) {
      if (!has_regions) return true;
      for (int32_t q = P.part_hex_start[p]; q < P.part_hex_start[p] + P.part_hex_count[p]; ++q)
        if (P.hex_slot_elem[q] >= 0 && o.element_region[P.hex_slot_elem[q]] != 0) return false;
      for (int32_t q = P.part_tet_start[p]; q < P.part_tet_start[p] + P.part_tet_count[p]; ++q)
        if (P.tet_slot_elem[q] >= 0 && o.element_region[P.tet_slot_elem[q]] != 0) return false;
      return true;
    };
    if (ok) {
      auto first = plist.begin() + st->n_boundary + st->n_mixed_i;
      auto mid = std::stable_partition(first, plist.end(),
                                       [&](int32_t p) { return !(P.part_tet_count[p] == 0 && region0(p)); });
      st->n_lean_i = (int)(plist.end() - mid);
      // tets in colour phases with one accumulator row and plain 14-bit node references
      if (P.colored_ok && P.tet_rows == 1 && P.max_local_nodes + 1 < (1 << 14)) {
        auto mfirst = plist.begin() + st->n_boundary;
        auto mmid = std::stable_partition(mfirst, mfirst + st->n_mixed_i, [&](int32_t p) { return !region0(p); });
        st->n_lean_mixed_i = (int)((mfirst + st->n_mixed_i) - mmid);
      }
    }
  }
  st->part_list.upload(plist, s);
  if (e->X.world > 1) {
    e->x_send.upload(e->X.send_nodes, s);
    e->x_recv.upload(e->X.recv_nodes, s);
    e->x_sendbuf.alloc(sizeof(S) * std::max<size_t>(1, e->X.send_nodes.size()));
    e->x_recvbuf.alloc(sizeof(S) * std::max<size_t>(1, e->X.recv_nodes.size()));
    FH_CUDA(cudaStreamCreateWithFlags(&e->comm_stream, cudaStreamNonBlocking));
    FH_CUDA(cudaEventCreateWithFlags(&e->ev_packed, cudaEventDisableTiming));
    FH_CUDA(cudaEventCreateWithFlags(&e->ev_halo, cudaEventDisableTiming));
  }
  std::vector<int32_t> robin_base(P.n_parts + 1, 0);
  for (int p = 0; p < P.n_parts; ++p) robin_base[p + 1] = robin_base[p] + (P.part_n_free[p] - P.part_robin_start[p]);
  st->part_node_start.upload(P.part_node_start, s);
  st->part_n_free.upload(P.part_n_free, s);
  st->part_robin_start.upload(P.part_robin_start, s);
  st->part_robin_base.upload(robin_base, s);
  st->part_tet_start.upload(P.part_tet_start, s);
  st->part_hex_start.upload(P.part_hex_start, s);
  st->part_tet_count.upload(P.part_tet_count, s);
  st->part_hex_count.upload(P.part_hex_count, s);
  st->part_halo_start.upload(P.part_halo_start, s);
  {  // +4 entries: the kernel bulk-copies each tile's list widened to 16-byte boundaries
    std::vector<int32_t> hn(P.halo_nodes);
    hn.resize(hn.size() + 4, 0);
    st->halo_nodes.upload(hn, s);
  }
  if (!e->td) {  // the TI freeze kernel works on global ids
    st->tet_conn.upload(P.tet_conn, s);
    st->hex_conn.upload(P.hex_conn, s);
  }
  st->tet_slot_elem.upload(P.tet_slot_elem, s);
  st->hex_slot_elem.upload(P.hex_slot_elem, s);
  // accumulation mode (fh_tiled.cu): colour phases when the colouring fits,
  // else ranked phases; FH_TILE_MODE (0..3) overrides (tuning knob)
  // measured (scripts/sweep.py): corner phases win on corner-unique hex grids (cfg4),
  // colour phases win on tets (cfg3, 1.45x over ranked)
  const bool hex_colour_ok = P.colored_ok && P.hex_colored;
  // fp32 corner-unique hexes: two accumulator rows (4 barriers/batch) measured
  // 1% faster than one row; fp64 keeps one row (shared memory)
  const int corner_mode = sizeof(S) == 4 ? kModeCornerPhase2 : kModeCornerPhase;
  int mode = P.corner_unique ? corner_mode : (hex_colour_ok ? kModeColored : kModeRanked);
  if (o.tile_mode > 0) {  // fh_options.tile_mode = mode + 1 (explicit, checked)
    const int m = o.tile_mode - 1;
    if (m == kModeSharedAtomic && !o.allow_nondeterministic)
      fail(FH_ERR_CONFIG, "tile_mode shared-memory atomics is non-deterministic: set allow_nondeterministic");
    if (m == kModeRanked || m == kModeSharedAtomic || (m == kModeColored && hex_colour_ok) ||
        ((m == kModeCornerPhase || m == kModeCornerPhase2) &&
         P.corner_unique))
      mode = m;
    else
      fail(FH_ERR_CONFIG, "tile_mode " + std::to_string(o.tile_mode) + " does not apply to this mesh");
  }
  // `mode` is the hex mode (kernel template); tets never are corner-unique and
  // always use colour phases (or ranked phases if the colouring overflowed)
  const int tet_mode = P.colored_ok ? kModeColored : kModeRanked;
  if (mode == kModeRanked) st->hex_rank.upload(P.hex_rank, s);
  if (tet_mode == kModeRanked) st->tet_rank.upload(P.tet_rank, s);
  if (mode == kModeColored) {
    st->hex_phase.upload(P.hex_phase, s);
    st->hex_bnph.upload(P.hex_batch_nph, s);
  }
  if (tet_mode == kModeColored) {
    st->tet_phase.upload(P.tet_phase, s);
    st->tet_bnph.upload(P.tet_batch_nph, s);
  }
  const int64_t nts = (int64_t)P.tet_slot_elem.size(), nhs = (int64_t)P.hex_slot_elem.size();
  // batch records: the 16-bit connectivity goes in by a pitched copy, G by k_pack_slots
  auto make_rec = [&](DBuf<unsigned char> &rec, const std::vector<uint16_t> &conn16, int64_t n, int N) {
    const int64_t nbat = n / kBatch;  // slot ranges are batch-padded
    rec.alloc((size_t)nbat * RecBytes<S>(N));
    if (nbat)
      FH_CUDA(cudaMemcpy2DAsync(rec.p, RecBytes<S>(N), conn16.data(), (size_t)kBatch * N * 2, (size_t)kBatch * N * 2,
                                (size_t)nbat, cudaMemcpyHostToDevice, s));
  };
  make_rec(st->tet_rec, P.tet_conn16, nts, 4);
  make_rec(st->hex_rec, P.hex_conn16, nhs, 8);
  const bool regions = o.n_materials > 1 && o.element_region;
  if (e->kfactor.p && !e->td) {  // TD: folded into G by k_pack_slots
    st->tet_kf.alloc(nts);
    st->hex_kf.alloc(nhs);
  }
  if (regions) {
    st->tet_region.alloc(nts);
    st->hex_region.alloc(nhs);
    // tiles whose slots all lie in one region skip the per-slot region bytes
    std::vector<int8_t> pr(P.n_parts);
    for (int p = 0; p < P.n_parts; ++p) {
      int r = -2;
      auto scan = [&](const std::vector<int32_t> &slot_elem, int32_t start, int32_t count) {
        for (int32_t q = start; q < start + count && r != -1; ++q) {
          const int32_t el = slot_elem[q];
          if (el < 0) continue;
          const int re = o.element_region[el];
          r = (r == -2 || r == re) ? re : -1;
        }
      };
      scan(P.tet_slot_elem, P.part_tet_start[p], P.part_tet_count[p]);
      scan(P.hex_slot_elem, P.part_hex_start[p], P.part_hex_count[p]);
      pr[p] = (int8_t)(r < 0 || r > 127 ? -1 : r);
    }
    st->part_region.upload(pr, s);
  }
  // LEAN batch loops (fh_tiled.cu): tet-only colour tiles with 4 rows or
  // hex-only two-row corner-phase tiles, one material, TD two-knot laws, no
  // kf stream, <= 256 batches per tile.  Their fp32
  // records store G as 3 interleaved pairs (one 8-byte load per pair; the
  // 16-byte fp64 pairs measured 1.4% slower on cfg3, so fp64 keeps 6 rows).
  {
    MatSet<S> mt = mats_of<S>(e);
    const bool lin_ok = normalise_curves(mt) != 0;
    int max_b = 0;
    for (int q = 0; q < P.n_parts; ++q)
      max_b = std::max(max_b, (P.part_tet_count[q] + kBatch - 1) / kBatch + (P.part_hex_count[q] + kBatch - 1) / kBatch);
    const bool kind_ok = nhs == 0 ? (tet_mode == kModeColored && P.tet_rows >= 2)
                                  : (nts == 0 && mode == kModeCornerPhase2);
    // fp32 LEAN records hold byte offsets in 16 (hex) / 14 (tets) bits
    const bool offs_ok = sizeof(S) != 4 || 4 * ((int64_t)P.max_local_nodes + 1) <= (nhs == 0 ? 0x3fff : 0xffff);
    st->lean = e->td && lin_ok && o.lean_kernels == 0 && !regions &&
               !st->tet_kf.p && !st->hex_kf.p && kind_ok && max_b <= kBatch && offs_ok;
    if (st->lean && sizeof(S) == 4) {
      if (nts)
        k_scale_conn<<<nblk(nts * 4), kBlk, 0, s>>>(st->tet_rec.p, nts / kBatch, RecBytes<S>(4), kBatch * 4, 1);
      if (nhs)
        k_scale_conn<<<nblk(nhs * 8), kBlk, 0, s>>>(st->hex_rec.p, nhs / kBatch, RecBytes<S>(8), kBatch * 8, 0);
    }
  }
  if (nts)
    k_pack_slots<S><<<nblk(nts), kBlk, 0, s>>>(st->tet_slot_elem.p, nts, G_dev, 1.0,
                                               reinterpret_cast<S *>(st->tet_rec.p), RecBytes<S>(4) / (int)sizeof(S),
                                               kBatch * 4 * 2 / (int)sizeof(S), e->kfactor.p, st->tet_kf.p,
                                               e->elem_region.p, st->tet_region.p, st->lean && sizeof(S) == 4);
  if (nhs)
    k_pack_slots<S><<<nblk(nhs), kBlk, 0, s>>>(st->hex_slot_elem.p, nhs, G_dev, 1.0 / 64.0,
                                               reinterpret_cast<S *>(st->hex_rec.p), RecBytes<S>(8) / (int)sizeof(S),
                                               kBatch * 8 * 2 / (int)sizeof(S), e->kfactor.p, st->hex_kf.p,
                                               e->elem_region.p, st->hex_region.p, st->lean && sizeof(S) == 4);
  FH_CUDA(cudaGetLastError());
  // nodal arrays in the new (multi-GPU: rank-local) numbering
  st->T[0].alloc(Vt);
  st->T[1].alloc(Vt);
  st->vol.alloc(Vt);
  {
    float *vf = nullptr;
    double *vd = nullptr;
    if constexpr (sizeof(S) == 4) vf = st->vol.p; else vd = st->vol.p;
    k_to_new<<<nblk(Vt), kBlk, 0, s>>>(e->node_vol.p, e->old_of_new.p, Vt, vf, vd, nullptr, nullptr);
  }
  if (regions) {
    std::vector<int32_t> nr(V);
    FH_CUDA(cudaMemcpyAsync(nr.data(), e->node_region.p, sizeof(int32_t) * V, cudaMemcpyDeviceToHost, s));
    FH_CUDA(cudaStreamSynchronize(s));
    std::vector<uint8_t> nrn(Vt);
    for (int64_t n = 0; n < Vt; ++n) nrn[n] = (uint8_t)nr[P.old_of_new[n]];
    st->node_region.upload(nrn, s);
    // per tile: the material of its updated nodes when they all share one
    // (the node update then reads the laws as uniform operands), else -1
    std::vector<int8_t> pm(P.n_parts);
    for (int p = 0; p < P.n_parts; ++p) {
      const int64_t a = P.part_node_start[p], b = a + P.part_n_free[p];
      int m = b > a ? nrn[a] : 0;
      for (int64_t n = a; n < b && m >= 0; ++n)
        if (nrn[n] != m) m = -1;
      pm[p] = (int8_t)m;
    }
    st->part_mat.upload(pm, s);
  }
  if (!e->td) {
    st->cap.alloc(Vt);
    st->kb.alloc(Vt);
    st->tet_kbar.alloc(nts);
    st->hex_kbar.alloc(nhs);
  }
  if (!e->q_static.empty() || !e->load_power.empty()) {
    st->q_ext.alloc(Vt);
    if (e->load_power.empty()) {
      FH_CUDA(cudaMemcpyAsync(e->stage.p, e->q_static.data(), sizeof(double) * V, cudaMemcpyHostToDevice, s));
      float *qf = nullptr;
      double *qd = nullptr;
      if constexpr (sizeof(S) == 4) qf = st->q_ext.p; else qd = st->q_ext.p;
      k_to_new<<<nblk(Vt), kBlk, 0, s>>>(e->stage.p, e->old_of_new.p, Vt, qf, qd, nullptr, nullptr);
    }
  }
  if (!e->sources.empty()) {
    st->xyz.alloc(4 * Vt);
    k_xyzv_to_new<S><<<nblk(Vt), kBlk, 0, s>>>(e->xyz.p, e->old_of_new.p, st->vol.p, Vt, st->xyz.p);
    FH_CUDA(cudaGetLastError());
  }
  if (!e->robin_nodes.empty()) {
    // compact robin arrays ordered like the renumbered robin nodes
    std::vector<int64_t> slot_of(V, -1);
    for (size_t q = 0; q < e->robin_nodes.size(); ++q) slot_of[e->robin_nodes[q]] = (int64_t)q;
    std::vector<S> ha(robin_base[P.n_parts]), hat(robin_base[P.n_parts]);
    for (int p = 0; p < P.n_parts; ++p)
      for (int loc = P.part_robin_start[p]; loc < P.part_n_free[p]; ++loc) {
        const int64_t q = slot_of[P.old_of_new[P.part_node_start[p] + loc]];
        ha[robin_base[p] + loc - P.part_robin_start[p]] = (S)e->robin_hA[q];
        hat[robin_base[p] + loc - P.part_robin_start[p]] = (S)e->robin_hAT[q];
      }
    st->robin_hA.upload(ha, s);
    st->robin_hAT.upload(hat, s);
  }
  if (!e->dir_nodes.empty()) {  // imposed on the device whenever a field is set (solver.py:364-365)
    std::vector<int32_t> ids;
    std::vector<S> vals;
    for (size_t q = 0; q < e->dir_nodes.size(); ++q) {
      const int64_t l = P.new_of_old[e->dir_nodes[q]];
      if (l < 0) continue;  // not in this rank's view
      ids.push_back((int32_t)l);
      vals.push_back((S)e->dir_vals[q]);
    }
    st->dir_ids.upload(ids, s);
    st->dir_vals.upload(vals, s);
  }
  g.part_list = st->part_list.p;
  g.part_node_start = st->part_node_start.p;
  g.part_n_free = st->part_n_free.p;
  g.part_robin_start = st->part_robin_start.p;
  g.part_robin_base = st->part_robin_base.p;
  g.part_tet_start = st->part_tet_start.p;
  g.part_hex_start = st->part_hex_start.p;
  g.part_tet_count = st->part_tet_count.p;
  g.part_hex_count = st->part_hex_count.p;
  g.part_halo_start = st->part_halo_start.p;
  g.halo_nodes = st->halo_nodes.p;
  g.tet_rec = st->tet_rec.p;
  g.hex_rec = st->hex_rec.p;
  g.tet_kf = st->tet_kf.p;
  g.hex_kf = st->hex_kf.p;
  g.tet_phase = st->tet_phase.p;
  g.hex_phase = st->hex_phase.p;
  g.tet_bnph = st->tet_bnph.p;
  g.hex_bnph = st->hex_bnph.p;
  g.tet_rank = st->tet_rank.p;
  g.hex_rank = st->hex_rank.p;
  g.tet_region = st->tet_region.p;
  g.hex_region = st->hex_region.p;
  g.max_phase_tet = P.max_phase_tet;
  g.max_phase_hex = P.max_phase_hex;
  g.vol = st->vol.p;
  g.cap_frozen = st->cap.p;
  g.kb_frozen = st->kb.p;
  g.q_ext = st->q_ext.p;
  g.xyzv = st->xyz.p;
  g.node_region = st->node_region.p;
  g.part_mat = st->part_mat.p;
  g.part_region = st->part_region.p;
  g.robin_hA = st->robin_hA.p;
  g.robin_hAT = st->robin_hAT.p;
  g.mats = mats_of<S>(e);
  g.lin = normalise_curves(g.mats);
  g.lin_lo = -std::numeric_limits<S>::infinity();
  g.lin_hi = std::numeric_limits<S>::infinity();
  if (g.lin) {
    const Mat<S> &m0 = g.mats.m[0];
    const Curve<S> *cs[4] = {&m0.rho, &m0.c, &m0.k, m0.td_perf ? &m0.wb : nullptr};
    for (const Curve<S> *c : cs)
      if (c && c->n == 2 && c->slope[0] != S(0)) {
        g.lin_lo = std::max(g.lin_lo, c->x[0]);
        g.lin_hi = std::min(g.lin_hi, c->x[1]);
      }
  }
  g.tet_rows = P.tet_rows;
  g.n_src = 0;  // set per step from the active sources
  g.n_gauss = 0;
  g.runaway_limit = (S)e->runaway_limit;
  g.flag = e->flag.p;
  g.n_nodes = Vt;
  g.lean = st->lean ? 1 : 0;
  g.max_tile_batches = 0;
  for (int q = 0; q < P.n_parts; ++q)
    g.max_tile_batches = std::max(g.max_tile_batches, (P.part_tet_count[q] + kBatch - 1) / kBatch +
                                                          (P.part_hex_count[q] + kBatch - 1) / kBatch);
  g.max_local = std::max(1, P.max_local_nodes);
  auto al = [](size_t b) { return (b + 127) & ~(size_t)127; };
  // accumulation mode: corner phases / corner slots need corner-unique tiles;
  // FH_TILE_MODE (0/1/2) and FH_TILE_STAGES override the defaults (tuning knobs)
  st->mode = mode;
  g.n_stages = 2;  // measured best on cfg4 (scripts/sweep.py)
  if (o.tile_stages > 0) g.n_stages = std::min(kMaxStages, o.tile_stages);
  // +1: the dummy node the padding slots point at (partition step 5)
  // staged per node: T, plus k(T) only for laws with more than two knots (fh_tiled.cu, Staged)
  // (+4: the owned range is bulk-copied from the 16-byte boundary below its first node)
  g.smem_T = (int)al((e->td && !g.lin ? 2 : 1) * sizeof(S) * ((size_t)std::max(1, P.max_local_nodes) + 1 + 4));
  // +1: the trash slot of the corner-phase accumulation
  const int rows = std::max(st->mode == kModeCornerPhase2 ? 2 : 1,
                            P.tet_rows);
  g.smem_acc = (int)al(sizeof(S) * rows * ((size_t)std::max(1, P.max_part_free) + 1));
  {  // the accumulator region first holds the tile's halo id list (bulk copy)
    int max_halo = 0;
    for (int q = 0; q < P.n_parts; ++q) max_halo = std::max(max_halo, P.part_halo_start[q + 1] - P.part_halo_start[q]);
    g.smem_acc = std::max(g.smem_acc, (int)al(4 * ((size_t)max_halo + 8)));
  }
  int stage = 0;
  if (e->n_tet)
    stage = std::max(stage, StageBytes<S>(4, st->tet_kf.p || !e->td, tet_mode == kModeRanked, tet_mode == kModeColored,
                                          st->tet_region.p != nullptr));
  if (e->n_hex)
    stage = std::max(stage, StageBytes<S>(8, st->hex_kf.p || !e->td, mode == kModeRanked, mode == kModeColored,
                                          st->hex_region.p != nullptr));
  g.stage_bytes = (int)al(stage);
  st->smem = (size_t)g.smem_T + g.smem_acc + (size_t)g.n_stages * g.stage_bytes;
  if (st->smem > 220 * 1024) fail(FH_ERR_CONFIG, "tile too large for shared memory; lower part_nodes");
  // wave fit, second pass: the first pass assumed the launch bounds' CTAs per
  // SM; if the kernel actually keeps a different number resident at this
  // shared memory size (fp64 tiles), partition again for that count
  if (o.part_nodes <= 0 && e->refit_per_sm == 0 && !(V / target_used < 2 * 148)) {
    const int bps = tiled_occupancy<S>(g, e->td, mode, st->smem);
    if (bps > 0 && wave_fit_part_nodes(default_part_nodes(sizeof(S) == 4 ? 32 : 64, e->n_tet, e->n_hex), V,
                                       std::max(1, o.n_domains), sizeof(S) == 4 ? 32 : 64, e->n_tet, e->n_hex,
                                       o.device, bps) != target_used) {
      e->refit_per_sm = bps;
      FH_CUDA(cudaStreamSynchronize(s));
      setup_tiled<S>(e, mesh, b, G_dev);  // replaces the partition and every tiled buffer
      return;
    }
  }
  FH_CUDA(cudaStreamSynchronize(s));
  if constexpr (sizeof(S) == 4)
    e->tf = std::move(st);
  else
    e->tdd = std::move(st);
}

// ATOMIC: element streams (sorted by smallest new node id), G SoA, node classes
template <typename S>
void setup_atomic(fh_engine *e, const fh_mesh &mesh, const double *G_dev) {
  cudaStream_t s = e->stream;
  const Partition &P = e->part;
  auto build = [&](const int64_t *conn, int64_t n, int N, int64_t e0, double scale, DBuf<int32_t> &dconn,
                   DBuf<char> &dG) {
    if (n == 0) return;
    std::vector<int32_t> order(n);
    std::vector<int64_t> key(n);
    for (int64_t i = 0; i < n; ++i) {
      int64_t k = INT64_MAX;
      for (int a = 0; a < N; ++a) k = std::min<int64_t>(k, P.new_of_old[conn[N * i + a]]);
      key[i] = k;
      order[i] = (int32_t)i;
    }
    std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return key[x] < key[y]; });
    std::vector<int32_t> c((size_t)N * n), elem(n);
    for (int64_t i = 0; i < n; ++i) {
      elem[i] = (int32_t)(e0 + order[i]);
      for (int a = 0; a < N; ++a) c[(size_t)N * i + a] = (int32_t)P.new_of_old[conn[N * (int64_t)order[i] + a]];
    }
    dconn.upload(c, s);
    DBuf<int32_t> delem;
    delem.upload(elem, s);
    dG.alloc(6 * sizeof(S) * (size_t)n);
    atomic_pack<S>(delem.p, n, G_dev, scale, e->kfactor.p, reinterpret_cast<S *>(dG.p), s);
    FH_CUDA(cudaStreamSynchronize(s));
  };
  build(mesh.tets, e->n_tet, 4, 0, 1.0, e->a_tet_conn, e->a_tet_G);
  build(mesh.hexes, e->n_hex, 8, e->n_tet, 1.0 / 64.0, e->a_hex_conn, e->a_hex_G);
  std::vector<uint8_t> cls(e->Vt, 0);
  for (int p = 0; p < P.n_parts; ++p)
    for (int32_t n = P.part_node_start[p] + P.part_n_free[p]; n < P.part_node_start[p + 1]; ++n) cls[n] = 2;
  if (!e->robin_nodes.empty()) {
    std::vector<S> ha(e->Vt, S(0)), hat(e->Vt, S(0));
    for (size_t q = 0; q < e->robin_nodes.size(); ++q) {
      const int64_t n = P.new_of_old[e->robin_nodes[q]];
      if (n < 0 || cls[n] == 2) continue;  // Dirichlet wins
      cls[n] = 1;
      ha[n] = (S)e->robin_hA[q];
      hat[n] = (S)e->robin_hAT[q];
    }
    e->a_hA.alloc(sizeof(S) * (size_t)e->Vt);
    e->a_hAT.alloc(sizeof(S) * (size_t)e->Vt);
    FH_CUDA(cudaMemcpyAsync(e->a_hA.p, ha.data(), sizeof(S) * e->Vt, cudaMemcpyHostToDevice, s));
    FH_CUDA(cudaMemcpyAsync(e->a_hAT.p, hat.data(), sizeof(S) * e->Vt, cudaMemcpyHostToDevice, s));
    FH_CUDA(cudaStreamSynchronize(s));
    e->atom.hA = e->a_hA.p;
    e->atom.hAT = e->a_hAT.p;
  }
  e->a_cls.upload(cls, s);
  e->a_F.alloc(sizeof(S) * (size_t)e->Vt);
  e->a_F.zero(s);
  AtomicState &a = e->atom;
  a.tet_conn = e->a_tet_conn.p;
  a.hex_conn = e->a_hex_conn.p;
  a.tet_G = e->a_tet_G.p;
  a.hex_G = e->a_hex_G.p;
  a.n_tet = e->n_tet;
  a.n_hex = e->n_hex;
  a.V = e->Vt;
  a.cls = e->a_cls.p;
  FH_CUDA(cudaStreamSynchronize(s));
}

template <typename S>
void tiled_set_T(fh_engine *e, const double *src = nullptr) {  // src (default e->stage): original order
  TiledState<S> &st = tstate<S>(e);
  float *f0 = nullptr, *f1 = nullptr;
  double *d0 = nullptr, *d1 = nullptr;
  if constexpr (sizeof(S) == 4) {
    f0 = st.T[0].p;
    f1 = st.T[1].p;
  } else {
    d0 = st.T[0].p;
    d1 = st.T[1].p;
  }
  k_to_new<<<nblk(e->Vt), kBlk, 0, e->stream>>>(src ? src : e->stage.p, e->old_of_new.p, e->Vt, f0, d0, f1, d1);
  // the reference steps from the state as given and imposes the Dirichlet
  // values after the update (solver.py:364-365): the first step reads T[0]
  // as set and writes T[1], which already holds the Dirichlet values (the
  // kernel never writes those nodes); T[0] gets them right after that step
  if (st.dir_ids.n)
    k_scatter_dir<S><<<nblk((int64_t)st.dir_ids.n), kBlk, 0, e->stream>>>(st.T[1].p, st.dir_ids.p,
                                                                         st.dir_vals.p, (int64_t)st.dir_ids.n);
  st.dir_pending = st.dir_ids.n > 0;
  FH_CUDA(cudaGetLastError());
  st.cur = 0;
}

template <typename S>
void tiled_get_T(fh_engine *e, double *dst_dev) {
  TiledState<S> &st = tstate<S>(e);
  k_to_old<S><<<nblk(e->V), kBlk, 0, e->stream>>>(st.T[st.cur].p, e->new_of_old.p, e->V, dst_dev);
  FH_CUDA(cudaGetLastError());
}

// current field, original order, fp64, into dst (default e->stage; device)
void current_T_to_stage(fh_engine *e, double *dst = nullptr) {
  double *d = dst ? dst : e->stage.p;
  if (e->assembly == FH_ASSEMBLY_EXACT) {
    FH_CUDA(cudaMemcpyAsync(d, e->T.p, sizeof(double) * e->V, cudaMemcpyDeviceToDevice, e->stream));
  } else if (e->precision == 32) {
    tiled_get_T<float>(e, d);
  } else {
    tiled_get_T<double>(e, d);
  }
}

template <typename S>
void tiled_run(fh_engine *e, int64_t nsteps, double dt) {
  TiledState<S> &st = tstate<S>(e);
  TiledArgs<S> &g = st.args;
  const int64_t step0 = e->step_index;
  for (int64_t k = 0; k < nsteps; ++k) {
    const double t = e->time;
    upload_qr(e, t);
    g.Tin = st.T[st.cur].p;
    g.Tout = st.T[st.cur ^ 1].p;
    if (!e->td && !e->frozen) {
      const int64_t nts = (int64_t)e->part.tet_slot_elem.size(), nhs = (int64_t)e->part.hex_slot_elem.size();
      tiled_freeze<S>(g, st.tet_conn.p, st.hex_conn.p, nts, nhs, e->Vt, st.tet_kf.p, st.hex_kf.p, st.tet_kbar.p, st.hex_kbar.p, st.cap.p,
                      st.kb.p, e->stream);
      g.tet_kf = st.tet_kbar.p;
      g.hex_kf = st.hex_kbar.p;
      e->frozen = true;
    }
    g.dt = (S)dt;
    g.step_no = (unsigned long long)(e->step_index + 1);
    g.F_out = e->keep_inflow ? st.F.p : nullptr;
    // active sources only, Gaussians first (the kernel loops over each kind
    // without per-source branches)
    int ns = 0;
    for (int pass = 0; pass < 2; ++pass) {
      for (const fh_source &src : e->sources) {
        if ((src.kind == FH_SOURCE_GAUSSIAN) != (pass == 0) || !(src.t0 <= t && t < src.t1)) continue;
        SourceT<S> &d = g.src[ns++];
        d.kind = src.kind;
        d.active = 1;
        d.amp = (S)src.amp;
        d.inv2s2 = (S)(1.0 / (2.0 * src.sigma * src.sigma));
        d.cap = (S)src.cap;
        d.inv4pi_amp = (S)(src.amp / (4.0 * M_PI));
        d.cx = (S)(src.x0[0] + src.vel[0] * t);
        d.cy = (S)(src.x0[1] + src.vel[1] * t);
        d.cz = (S)(src.x0[2] + src.vel[2] * t);
      }
      if (pass == 0) g.n_gauss = ns;
    }
    g.n_src = ns;
    // the tiles [begin, begin + count) of part_list: the first n_mixed hold
    // tets (mixed kernel), the rest only hexes (hex-only kernel instance)
    auto launch = [&](int begin, int count, int n_mixed) {
      g.part_begin = begin;
      if (n_mixed == count) {
        tiled_step(g, count, e->td, st.mode, st.smem, e->stream);
        return;
      }
      // the two instances run concurrently (disjoint tiles): the mixed tiles
      // on a side stream, so their last wave overlaps the hex-only tiles
      if (!e->kind_stream) {
        // highest priority: the side stream's few tiles are placed as SM slots free up, ahead of
        // the engine stream's many, so the step ends on the big launch's full-occupancy tail
        int prio_lo = 0, prio_hi = 0;
        FH_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        FH_CUDA(cudaStreamCreateWithPriority(&e->kind_stream, cudaStreamNonBlocking, prio_hi));
        FH_CUDA(cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming));
        FH_CUDA(cudaEventCreateWithFlags(&e->ev_join, cudaEventDisableTiming));
      }
      FH_CUDA(cudaEventRecord(e->ev_fork, e->stream));
      FH_CUDA(cudaStreamWaitEvent(e->kind_stream, e->ev_fork, 0));
      // the material-0 mixed tiles (end of the mixed range) run the LEAN 3 loop
      const int n_lm = (e->X.world == 1 && begin == st.n_boundary) ? std::min(st.n_lean_mixed_i, n_mixed) : 0;
      tiled_step(g, n_mixed - n_lm, e->td, st.mode, st.smem, e->kind_stream);
      if (n_lm > 0) {
        TiledArgs<S> gm = g;
        gm.part_begin = begin + n_mixed - n_lm;
        gm.lean = 3;
        tiled_step(gm, n_lm, e->td, st.mode, st.smem, e->kind_stream);
      }
      FH_CUDA(cudaEventRecord(e->ev_join, e->kind_stream));
      TiledArgs<S> gh = g;
      gh.tet_rec = nullptr;
      gh.part_begin = begin + n_mixed;
      const int n_lean = (e->X.world == 1) ? st.n_lean_i : 0;
      if (n_lean > 0) {  // material-0 hex tiles: LEAN 2 on the engine stream; the rest beside the mixed tiles
        if (count - n_mixed - n_lean > 0) {
          tiled_step(gh, count - n_mixed - n_lean, e->td, st.mode, st.smem, e->kind_stream);
          FH_CUDA(cudaEventRecord(e->ev_join, e->kind_stream));
        }
        TiledArgs<S> gl = gh;
        gl.part_begin = begin + count - n_lean;
        gl.lean = 2;
        tiled_step(gl, n_lean, e->td, st.mode, st.smem, e->stream);
      } else {
        tiled_step(gh, count - n_mixed, e->td, st.mode, st.smem, e->stream);
      }
      FH_CUDA(cudaStreamWaitEvent(e->stream, e->ev_join, 0));
    };
    if (e->assembly == FH_ASSEMBLY_ATOMIC) {
      atomic_step<S>(g, e->atom, reinterpret_cast<S *>(e->a_F.p), e->stream);
    } else if (e->X.world == 1) {
      launch(0, st.n_parts_local, st.n_mixed_i);
    } else {
      // interior tiles need no halo: they run while the previous step's
      // exchange is still in flight on the comm stream
      launch(st.n_boundary, st.n_parts_local - st.n_boundary, st.n_mixed_i);
      if (e->halo_pending) FH_CUDA(cudaStreamWaitEvent(e->stream, e->ev_halo, 0));
      e->halo_pending = false;
      launch(0, st.n_boundary, st.n_mixed_b);
      g.part_begin = 0;
      if (e->comm) {
        S *sendbuf = reinterpret_cast<S *>(e->x_sendbuf.p);
        S *recvbuf = reinterpret_cast<S *>(e->x_recvbuf.p);
        halo_pack<S>(g.Tout, e->x_send.p, (int64_t)e->X.send_nodes.size(), sendbuf, e->stream);
        FH_CUDA(cudaEventRecord(e->ev_packed, e->stream));
        FH_CUDA(cudaStreamWaitEvent(e->comm_stream, e->ev_packed, 0));
        nccl_exchange(e->comm, sendbuf, recvbuf, sizeof(S), e->X.peers, e->X.send_offs, e->X.recv_offs,
                      e->comm_stream);
        halo_unpack<S>(g.Tout, e->x_recv.p, (int64_t)e->X.recv_nodes.size(), recvbuf, e->comm_stream);
        FH_CUDA(cudaEventRecord(e->ev_halo, e->comm_stream));
        e->halo_pending = true;
      } else if (e->transport.exchange) {  // host transport: the same order, blocking exchange on the host
        S *sendbuf = reinterpret_cast<S *>(e->x_sendbuf.p);
        S *recvbuf = reinterpret_cast<S *>(e->x_recvbuf.p);
        const int64_t ns = (int64_t)e->X.send_nodes.size(), nr = (int64_t)e->X.recv_nodes.size();
        halo_pack<S>(g.Tout, e->x_send.p, ns, sendbuf, e->stream);
        e->x_host_send.resize(sizeof(S) * std::max<int64_t>(1, ns));
        e->x_host_recv.resize(sizeof(S) * std::max<int64_t>(1, nr));
        FH_CUDA(cudaMemcpyAsync(e->x_host_send.data(), sendbuf, sizeof(S) * ns, cudaMemcpyDeviceToHost, e->stream));
        FH_CUDA(cudaStreamSynchronize(e->stream));
        if (e->transport.exchange(e->transport.ctx, (int32_t)e->X.peers.size(), e->X.peers.data(),
                                  e->x_host_send.data(), e->X.send_offs.data(), e->x_host_recv.data(),
                                  e->X.recv_offs.data(), (int32_t)sizeof(S)) != 0)
          fail(FH_ERR_DEVICE, "host transport exchange failed");
        FH_CUDA(cudaMemcpyAsync(recvbuf, e->x_host_recv.data(), sizeof(S) * nr, cudaMemcpyHostToDevice, e->stream));
        halo_unpack<S>(g.Tout, e->x_recv.p, nr, recvbuf, e->stream);
      }
    }
    if (e->dir_runaway) k_flag_step<<<1, 1, 0, e->stream>>>(e->flag.p, g.step_no);
    if (st.dir_pending) {  // this step's input buffer is the next step's output
      k_scatter_dir<S><<<nblk((int64_t)st.dir_ids.n), kBlk, 0, e->stream>>>(
          st.T[st.cur].p, st.dir_ids.p, st.dir_vals.p, (int64_t)st.dir_ids.n);
      FH_CUDA(cudaGetLastError());
      st.dir_pending = false;
    }
    st.cur ^= 1;
    e->step_index += 1;
    e->time = (double)e->step_index * dt;
    if (e->n_probes && e->step_index % e->probe_interval == 0 && e->n_rec < e->probe_cap) {
      gather_probes_t<S>(st.T[st.cur].p, e->probes.p, e->n_probes, e->probe_hist.p + e->n_rec * e->n_probes,
                         e->flag.p, e->stream);
      e->probe_steps.push_back(e->step_index);
      e->n_rec++;
    }
  }
  (void)step0;
}

void exact_run(fh_engine *e, int64_t nsteps, double dt) {
  for (int64_t k = 0; k < nsteps; ++k) {
    const double t = e->time;
    upload_qr(e, t);
    if (!e->td && !e->frozen) {
      exact_props(e->ex, e->T.p, e->stream);
      e->frozen = true;
    }
    exact_step(e->ex, e->T.p, dt, t, e->step_index + 1, e->td, e->stream);
    if (e->dir_runaway) k_flag_step<<<1, 1, 0, e->stream>>>(e->flag.p, (unsigned long long)(e->step_index + 1));
    e->step_index += 1;
    e->time = (double)e->step_index * dt;
    if (e->n_probes && e->step_index % e->probe_interval == 0 && e->n_rec < e->probe_cap) {
      gather_probes(e->T.p, e->probes.p, e->n_probes, e->probe_hist.p + e->n_rec * e->n_probes, e->flag.p,
                    e->stream);
      e->probe_steps.push_back(e->step_index);
      e->n_rec++;
    }
  }
}

// would the active-load signature differ at step start time t?
bool loads_differ_at(const fh_engine *e, double t) {
  for (size_t l = 0; l < e->load_power.size(); ++l) {
    const uint8_t on = (e->load_t0[l] <= t && t < e->load_t1[l]);
    if (on != e->load_sig[l]) return true;
  }
  return false;
}

// EXACT on the resident kernel: one launch per segment of steps whose active
// loads do not change (q_r is re-uploaded between segments, as exact_run does
// before the step where a window opens or closes)
void resident_exact_run(fh_engine *e, int64_t nsteps, double dt) {
  int64_t k = 0;
  while (k < nsteps) {
    const double t = e->time;
    upload_qr(e, t);
    if (!e->td && !e->frozen) {
      exact_props(e->ex, e->T.p, e->stream);
      e->frozen = true;
    }
    int64_t seg = std::min<int64_t>(nsteps - k, (int64_t)1 << 30);
    if (!e->load_power.empty()) {
      seg = 1;
      while (k + seg < nsteps && seg < ((int64_t)1 << 30) && !loads_differ_at(e, (double)(e->step_index + seg) * dt))
        ++seg;
    }
    ResidentArgs r = e->res;
    if (r.ll[0]) {  // this launch's stamps: [epoch, epoch + seg]; never reused before the buffers are cleared
      if ((uint64_t)e->r_epoch + (uint64_t)seg + 1 >= 0xffffffffull) {
        e->r_ll[0].zero(e->stream);
        e->r_ll[1].zero(e->stream);
        e->r_epoch = 1;
      }
      r.stamp0 = e->r_epoch;
      e->r_epoch += (uint32_t)seg + 1u;
    }
    r.g = e->ex;
    r.step0 = e->step_index;
    r.nsteps = seg;
    r.time0 = t;
    r.dt = dt;
    r.probes = e->probes.p;
    r.n_probes = e->n_probes;
    r.probe_interval = e->probe_interval;
    r.rec0 = e->n_rec;
    r.rec_cap = e->probe_cap;
    r.probe_out = e->probe_hist.p;
    e->r_bar.zero(e->stream);
    resident_run(r, e->res_ctas, e->res_threads, e->res_smem, e->td, e->res_stage_k, e->stream);
    for (int64_t j = 0; j < seg; ++j) {  // the records the kernel writes (exact_run's bookkeeping)
      e->step_index += 1;
      if (e->n_probes && e->step_index % e->probe_interval == 0 && e->n_rec < e->probe_cap) {
        e->probe_steps.push_back(e->step_index);
        e->n_rec++;
      }
    }
    e->time = (double)e->step_index * dt;
    k += seg;
  }
}

void run_steps(fh_engine *e, int64_t nsteps, double dt) {
  if (e->assembly == FH_ASSEMBLY_EXACT && e->resident && !e->dir_runaway)
    resident_exact_run(e, nsteps, dt);
  else if (e->assembly == FH_ASSEMBLY_EXACT)
    exact_run(e, nsteps, dt);
  else if (e->precision == 32)
    tiled_run<float>(e, nsteps, dt);
  else
    tiled_run<double>(e, nsteps, dt);
}

// min over ranks of a host value (NCCL or the host transport; world 1: as is)
void rank_min_u64(fh_engine *e, unsigned long long &v) {
  if (e->comm) {
    if (!e->red_scratch.p) e->red_scratch.alloc(1);
    FH_CUDA(cudaMemcpyAsync(e->red_scratch.p, &v, sizeof(v), cudaMemcpyHostToDevice, e->stream));
    nccl_min_u64(e->comm, e->red_scratch.p, e->stream);
    FH_CUDA(cudaMemcpyAsync(&v, e->red_scratch.p, sizeof(v), cudaMemcpyDeviceToHost, e->stream));
    FH_CUDA(cudaStreamSynchronize(e->stream));
  } else if (e->transport.allreduce_min_u64) {
    uint64_t x = v;
    if (e->transport.allreduce_min_u64(e->transport.ctx, &x) != 0) fail(FH_ERR_DEVICE, "host transport all-reduce failed");
    v = x;
  }
}

bool multi_rank(const fh_engine *e) {
  return e->assembly != FH_ASSEMBLY_EXACT && e->X.world > 1 && (e->comm || e->transport.exchange);
}

// the field the next step reads, copied to / from e->snap (multi-GPU replay)
template <typename S>
void snapshot_T(fh_engine *e, bool restore) {
  TiledState<S> &st = tstate<S>(e);
  const size_t bytes = sizeof(S) * (size_t)e->Vt;
  if (!e->snap.p) e->snap.alloc(bytes);
  if (restore)
    FH_CUDA(cudaMemcpyAsync(st.T[st.cur].p, e->snap.p, bytes, cudaMemcpyDeviceToDevice, e->stream));
  else
    FH_CUDA(cudaMemcpyAsync(e->snap.p, st.T[st.cur].p, bytes, cudaMemcpyDeviceToDevice, e->stream));
}

// The instability report's node (solver.py:369-382: first non-finite node,
// else the first node of largest |T|) over this rank's owned nodes, agreed
// across ranks; returns the node (original id) and its value.
int64_t failure_node(fh_engine *e, double &value) {
  current_T_to_stage(e);
  std::vector<double> T(e->V);
  FH_CUDA(cudaMemcpyAsync(T.data(), e->stage.p, sizeof(double) * e->V, cudaMemcpyDeviceToHost, e->stream));
  FH_CUDA(cudaStreamSynchronize(e->stream));
  const bool multi = multi_rank(e);
  std::vector<int64_t> owned;  // original ids of the owned nodes, ascending
  if (multi) {
    owned.assign(e->part.old_of_new.begin() + e->X.node_lo, e->part.old_of_new.begin() + e->X.node_hi);
    std::sort(owned.begin(), owned.end());
  }
  const int64_t n_scan = multi ? (int64_t)owned.size() : e->V;
  auto id = [&](int64_t k) { return multi ? owned[k] : k; };
  const unsigned long long none = ~0ull;
  unsigned long long nf = none;
  for (int64_t k = 0; k < n_scan; ++k)
    if (!std::isfinite(T[id(k)])) {
      nf = (unsigned long long)id(k);
      break;
    }
  rank_min_u64(e, nf);
  int64_t node;
  if (nf != none) {
    node = (int64_t)nf;
  } else {
    double best = -1.0;
    int64_t arg = -1;
    for (int64_t k = 0; k < n_scan; ++k)
      if (std::fabs(T[id(k)]) > best) {
        best = std::fabs(T[id(k)]);
        arg = id(k);
      }
    // max |T| over ranks (non-negative doubles order like their bits), then
    // the lowest node id attaining it
    unsigned long long nb = ~(arg >= 0 ? (unsigned long long)__builtin_bit_cast(uint64_t, best) : 0ull);
    rank_min_u64(e, nb);
    unsigned long long cand = (arg >= 0 && ~nb == __builtin_bit_cast(uint64_t, best)) ? (unsigned long long)arg : none;
    rank_min_u64(e, cand);
    node = (int64_t)cand;
  }
  // the owning rank supplies the value
  bool mine = !multi || std::binary_search(owned.begin(), owned.end(), node);
  unsigned long long vb = mine ? __builtin_bit_cast(uint64_t, T[node]) : none;
  if (multi) rank_min_u64(e, vb);
  value = __builtin_bit_cast(double, (uint64_t)vb);
  return node;
}

int do_step(fh_engine *e, int64_t nsteps, double dt, fh_report *rep, float *elapsed_ms = nullptr,
            void *scratch = nullptr, size_t scratch_bytes = 0) {
  if (nsteps < 0) fail(FH_ERR_CONFIG, "nsteps must be >= 0");
  if (!(dt > 0.0) || !std::isfinite(dt)) fail(FH_ERR_CONFIG, "dt must be positive and finite");
  const int64_t step0 = e->step_index;
  const int cur0 = e->assembly == FH_ASSEMBLY_EXACT ? 0 : (e->precision == 32 ? e->tf->cur : e->tdd->cur);
  cudaEvent_t ev[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> sev;  // per-step start/stop events (L2-flushed timing)
  if (elapsed_ms && !scratch) {
    FH_CUDA(cudaEventCreate(&ev[0]));
    FH_CUDA(cudaEventCreate(&ev[1]));
    FH_CUDA(cudaEventRecord(ev[0], e->stream));
  }
  // multi-GPU: ranks that did not fail keep stepping until the call ends (the
  // flag is agreed once per call), so a failure is replayed from the field at
  // the start of the call for exactly the steps up to the failing one
  const bool multi = multi_rank(e);
  const int64_t nrec0 = e->n_rec;
  const size_t nps0 = e->probe_steps.size();
  const double time0 = e->time;
  bool dir_pending0 = false;
  if (multi) {
    if (e->precision == 32) {
      dir_pending0 = e->tf->dir_pending;
      snapshot_T<float>(e, false);
    } else {
      dir_pending0 = e->tdd->dir_pending;
      snapshot_T<double>(e, false);
    }
  }
  // resident EXACT kernel without a grid barrier: a runaway is only recorded
  // while the launch runs on, so the call is replayed from its start for
  // exactly the steps up to the failing one (deterministic; the field is then
  // the one right after that step, as on the two-launch path)
  const bool res_replay = e->assembly == FH_ASSEMBLY_EXACT && e->resident && !e->dir_runaway && e->res.ll[0];
  const bool frozen0 = e->frozen;
  if (res_replay)
    FH_CUDA(cudaMemcpyAsync(e->r_snap.p, e->T.p, sizeof(double) * (size_t)e->V, cudaMemcpyDeviceToDevice, e->stream));
  if (scratch) {
    sev.resize(2 * nsteps);
    for (auto &v : sev) FH_CUDA(cudaEventCreate(&v));
    for (int64_t k = 0; k < nsteps; ++k) {
      FH_CUDA(cudaMemsetAsync(scratch, (int)(k & 0xff), scratch_bytes, e->stream));
      FH_CUDA(cudaEventRecord(sev[2 * k], e->stream));
      run_steps(e, 1, dt);
      FH_CUDA(cudaEventRecord(sev[2 * k + 1], e->stream));
    }
  } else {
    run_steps(e, nsteps, dt);
  }
  if (scratch) {
    if (!sev.empty()) FH_CUDA(cudaEventSynchronize(sev.back()));
    float tot = 0.f;
    for (int64_t k = 0; k < nsteps; ++k) {
      float ms = 0.f;
      FH_CUDA(cudaEventElapsedTime(&ms, sev[2 * k], sev[2 * k + 1]));
      tot += ms;
    }
    for (auto &v : sev) cudaEventDestroy(v);
    if (elapsed_ms) *elapsed_ms = tot;
  }
  if (e->halo_pending) {  // the last step is complete once its halo has landed
    FH_CUDA(cudaStreamWaitEvent(e->stream, e->ev_halo, 0));
    e->halo_pending = false;
  }
  if (e->comm)  // every rank agrees on the first failing step
    nccl_min_u64(e->comm, &e->flag.p->step, e->stream);
  else if (e->transport.allreduce_min_u64) {
    FailFlag f0{};
    FH_CUDA(cudaMemcpyAsync(&f0, e->flag.p, sizeof(f0), cudaMemcpyDeviceToHost, e->stream));
    FH_CUDA(cudaStreamSynchronize(e->stream));
    rank_min_u64(e, f0.step);
    FH_CUDA(cudaMemcpyAsync(e->flag.p, &f0, sizeof(f0), cudaMemcpyHostToDevice, e->stream));
  }
  if (multi) {
    FailFlag fr{};
    FH_CUDA(cudaMemcpyAsync(&fr, e->flag.p, sizeof(fr), cudaMemcpyDeviceToHost, e->stream));
    FH_CUDA(cudaStreamSynchronize(e->stream));
    if (fr.step != ~0ull) {  // replay steps step0+1 .. fs from the snapshot on every rank
      const int64_t fs = (int64_t)fr.step;
      const FailFlag clear{~0ull};
      FH_CUDA(cudaMemcpyAsync(e->flag.p, &clear, sizeof(clear), cudaMemcpyHostToDevice, e->stream));
      if (e->precision == 32) {
        e->tf->cur = cur0;
        e->tf->dir_pending = dir_pending0;
        snapshot_T<float>(e, true);
      } else {
        e->tdd->cur = cur0;
        e->tdd->dir_pending = dir_pending0;
        snapshot_T<double>(e, true);
      }
      e->step_index = step0;
      e->time = time0;
      e->n_rec = nrec0;
      e->probe_steps.resize(nps0);
      e->qr_valid = false;
      run_steps(e, fs - step0, dt);
      if (e->halo_pending) {
        FH_CUDA(cudaStreamWaitEvent(e->stream, e->ev_halo, 0));
        e->halo_pending = false;
      }
      // the failing step ran again on its rank: the flag holds fs there
      if (e->comm) nccl_min_u64(e->comm, &e->flag.p->step, e->stream);
      else {
        FailFlag f1{};
        FH_CUDA(cudaMemcpyAsync(&f1, e->flag.p, sizeof(f1), cudaMemcpyDeviceToHost, e->stream));
        FH_CUDA(cudaStreamSynchronize(e->stream));
        rank_min_u64(e, f1.step);
        FH_CUDA(cudaMemcpyAsync(e->flag.p, &f1, sizeof(f1), cudaMemcpyHostToDevice, e->stream));
      }
    }
  }
  if (res_replay) {
    FailFlag fr{};
    unsigned long long lost = 0;
    FH_CUDA(cudaMemcpyAsync(&fr, e->flag.p, sizeof(fr), cudaMemcpyDeviceToHost, e->stream));
    FH_CUDA(cudaMemcpyAsync(&lost, e->r_bar.p, sizeof(lost), cudaMemcpyDeviceToHost, e->stream));
    FH_CUDA(cudaStreamSynchronize(e->stream));
    if (lost) fail(FH_ERR_DEVICE, "resident kernel: a CTA stopped receiving its neighbours' temperatures");
    if (fr.step != ~0ull && (int64_t)fr.step > step0) {
      const int64_t fs = (int64_t)fr.step;
      const FailFlag clear{~0ull};
      FH_CUDA(cudaMemcpyAsync(e->flag.p, &clear, sizeof(clear), cudaMemcpyHostToDevice, e->stream));
      FH_CUDA(cudaMemcpyAsync(e->T.p, e->r_snap.p, sizeof(double) * (size_t)e->V, cudaMemcpyDeviceToDevice, e->stream));
      e->step_index = step0;
      e->time = time0;
      e->n_rec = nrec0;
      e->probe_steps.resize(nps0);
      e->qr_valid = false;
      e->frozen = frozen0;
      run_steps(e, fs - step0, dt);  // its last step fails again and sets the flag to fs
    }
  }
  if (elapsed_ms && !scratch) {
    FH_CUDA(cudaEventRecord(ev[1], e->stream));
    FH_CUDA(cudaEventSynchronize(ev[1]));
    FH_CUDA(cudaEventElapsedTime(elapsed_ms, ev[0], ev[1]));
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
  }
  FailFlag f{};
  FH_CUDA(cudaMemcpyAsync(&f, e->flag.p, sizeof(f), cudaMemcpyDeviceToHost, e->stream));
  FH_CUDA(cudaStreamSynchronize(e->stream));
  if (rep) {
    std::memset(rep, 0, sizeof(*rep));
    rep->fail_step = -1;
    rep->fail_node = -1;
  }
  if (f.step != ~0ull) {
    const int64_t fs = (int64_t)f.step;
    // roll the host clock back to the failing step (later launches were no-ops)
    e->step_index = fs;
    e->time = (double)fs * dt;
    if (e->assembly != FH_ASSEMBLY_EXACT) {
      const int par = (int)((fs - step0) & 1);
      if (e->precision == 32) e->tf->cur = cur0 ^ par; else e->tdd->cur = cur0 ^ par;
    }
    while (!e->probe_steps.empty() && e->probe_steps.back() > fs) {
      e->probe_steps.pop_back();
      e->n_rec--;
    }
    // locate the node like solver.py:369-382 (first non-finite, else argmax |T|)
    double fail_value = 0.0;
    const int64_t node = failure_node(e, fail_value);
    if (rep) {
      rep->fail_step = fs;
      rep->fail_node = node;
      rep->fail_value = fail_value;
      rep->steps_done = fs - step0;
      rep->time = e->time;
      rep->step_index = e->step_index;
    }
    // clear the flag so the engine can be reused after set_temperature
    const FailFlag clear{~0ull};
    FH_CUDA(cudaMemcpy(e->flag.p, &clear, sizeof(clear), cudaMemcpyHostToDevice));
    g_last_error = "temperature at node " + std::to_string(node) + " is non-finite or beyond the runaway limit";
    return FH_ERR_INSTABILITY;
  }
  if (rep) {
    rep->steps_done = nsteps;
    rep->time = e->time;
    rep->step_index = e->step_index;
  }
  return FH_OK;
}

}  // namespace

// ============================================================================
extern "C" {

const char *fh_last_error(void) { return g_last_error.c_str(); }
int fh_version(void) { return 1; }

int fh_device_count(int *count) {
  FH_API_BEGIN
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
  *count = n;
  FH_API_END
}

int fh_create(const fh_mesh *mesh, const fh_boundary *bnd, const fh_options *opts, fh_engine **out) {
  FH_API_BEGIN
  if (!mesh || !bnd || !opts || !out) fail(FH_ERR_CONFIG, "null argument");
  *out = nullptr;
  auto e = std::make_unique<fh_engine>();
  e->opts = *opts;
  e->device = opts->device;
  e->precision = opts->precision == 32 ? 32 : 64;
  e->assembly = opts->assembly;
  e->td = opts->td_mode != 0;
  e->runaway_limit = opts->runaway_limit;
  if (e->assembly == FH_ASSEMBLY_EXACT && e->precision != 64) fail(FH_ERR_CONFIG, "EXACT mode is fp64 only");
  if (e->assembly != FH_ASSEMBLY_EXACT && e->assembly != FH_ASSEMBLY_TILED && e->assembly != FH_ASSEMBLY_ATOMIC)
    fail(FH_ERR_CONFIG, "unsupported assembly mode");
  if (e->assembly == FH_ASSEMBLY_ATOMIC) {
    if (!e->td) fail(FH_ERR_CONFIG, "ATOMIC assembly: temperature-dependent runs only");
    if (opts->n_materials > 1) fail(FH_ERR_CONFIG, "ATOMIC assembly: one material");
    if (opts->domain_hi > 0 && opts->domain_hi - std::max(0, opts->domain_lo) < std::max(1, opts->n_domains))
      fail(FH_ERR_CONFIG, "ATOMIC assembly: single GPU only");
  }
  e->V = mesh->n_nodes;
  e->n_tet = mesh->n_tets;
  e->n_hex = mesh->n_hexes;
  e->E = e->n_tet + e->n_hex;
  e->nconn = 4 * e->n_tet + 8 * e->n_hex;
  if (e->V <= 0 || e->E <= 0) fail(FH_ERR_CONFIG, "empty mesh");
  if (e->V >= (1ll << 31) || e->nconn >= (1ll << 31)) fail(FH_ERR_CONFIG, "mesh too large for 32-bit indices");
  fill_mats(e->mats_d, *opts);
  fill_mats(e->mats_f, *opts);
  FH_CUDA(cudaSetDevice(e->device));
  FH_CUDA(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
  cudaStream_t s = e->stream;
  // boundary (host copies)
  e->dir_nodes.assign(bnd->dirichlet_nodes, bnd->dirichlet_nodes + bnd->n_dirichlet);
  e->dir_vals.assign(bnd->dirichlet_values, bnd->dirichlet_values + bnd->n_dirichlet);
  for (int64_t i : e->dir_nodes)
    if (i < 0 || i >= e->V) fail(FH_ERR_CONFIG, "Dirichlet node out of range");
  for (double v : e->dir_vals)
    if (!(std::fabs(v) <= e->runaway_limit)) e->dir_runaway = true;
  if (bnd->n_loads > 0) {
    e->load_offs.assign(bnd->load_offsets, bnd->load_offsets + bnd->n_loads + 1);
    e->load_nodes.assign(bnd->load_nodes, bnd->load_nodes + e->load_offs.back());
    e->load_power.assign(bnd->load_power, bnd->load_power + bnd->n_loads);
    e->load_t0.assign(bnd->load_t0, bnd->load_t0 + bnd->n_loads);
    e->load_t1.assign(bnd->load_t1, bnd->load_t1 + bnd->n_loads);
    e->load_sig.assign(bnd->n_loads, 0);
  }
  if (bnd->q_static) e->q_static.assign(bnd->q_static, bnd->q_static + e->V);
  if (bnd->n_sources > kMaxSources) fail(FH_ERR_CONFIG, "too many sources");
  e->sources.assign(bnd->sources, bnd->sources + std::max(0, bnd->n_sources));
  if (bnd->n_robin > 0) {
    e->robin_nodes.assign(bnd->robin_nodes, bnd->robin_nodes + bnd->n_robin);
    e->robin_hA.assign(bnd->robin_hA, bnd->robin_hA + bnd->n_robin);
    e->robin_hAT.assign(bnd->robin_hAT, bnd->robin_hAT + bnd->n_robin);
  }
  // connectivity + CSR (host bookkeeping), device copies
  std::vector<int32_t> conn(e->nconn);
  for (int64_t p = 0; p < 4 * e->n_tet; ++p) conn[p] = (int32_t)mesh->tets[p];
  for (int64_t p = 0; p < 8 * e->n_hex; ++p) conn[4 * e->n_tet + p] = (int32_t)mesh->hexes[p];
  for (int32_t v : conn)
    if (v < 0 || v >= e->V) fail(FH_ERR_CONFIG, "element references a node out of range");
  std::vector<int32_t> offs, pos;
  build_node_csr(e->V, e->n_tet, mesh->tets, e->n_hex, mesh->hexes, offs, pos);
  e->conn.upload(conn, s);
  e->csr_offs.upload(offs, s);
  e->csr_pos.upload(pos, s);
  e->xyz.upload(mesh->coords, 3 * e->V, s);
  if (opts->element_kfactor) e->kfactor.upload(opts->element_kfactor, e->E, s);
  // regions: node region = largest region id among incident elements
  if (opts->n_materials > 1 && opts->element_region) {
    std::vector<int32_t> er(opts->element_region, opts->element_region + e->E), nr(e->V, 0);
    for (int32_t r : er)
      if (r < 0 || r >= opts->n_materials) fail(FH_ERR_CONFIG, "element region out of range");
    for (int64_t i = 0; i < e->V; ++i)
      for (int32_t q = offs[i]; q < offs[i + 1]; ++q) {
        const int64_t p = pos[q];
        const int64_t el = p < 4 * e->n_tet ? p / 4 : e->n_tet + (p - 4 * e->n_tet) / 8;
        nr[i] = std::max(nr[i], er[el]);
      }
    e->elem_region.upload(er, s);
    e->node_region.upload(nr, s);
  }
  // device precompute (fh_precompute.cu)
  e->elem_vol.alloc(e->E);
  e->node_vol.alloc(e->V);
  e->row_abs.alloc(e->nconn);
  DBuf<double> G;
  DBuf<int> bad;
  bad.alloc(1);
  const int big = 0x7fffffff;
  FH_CUDA(cudaMemcpyAsync(bad.p, &big, sizeof(int), cudaMemcpyHostToDevice, s));
  GeomOut go{};
  go.vol = e->elem_vol.p;
  go.row_abs = e->row_abs.p;
  go.bad = bad.p;
  if (e->assembly == FH_ASSEMBLY_EXACT) {
    e->A.alloc(16 * e->n_tet + 64 * e->n_hex);
    go.A = e->A.p;
  } else {
    G.alloc(6 * e->E);
    go.G = G.p;
  }
  launch_geometry(e->xyz.p, e->conn.p, e->n_tet, e->n_hex, go, s);
  int first_bad = big;
  FH_CUDA(cudaMemcpyAsync(&first_bad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  FH_CUDA(cudaStreamSynchronize(s));
  if (first_bad != big)
    fail(FH_ERR_DEGENERATE, "element " + std::to_string(first_bad) + ": non-positive volume / Jacobian");
  launch_node_volumes(e->csr_offs.p, e->csr_pos.p, e->V, e->n_tet, e->elem_vol.p, e->node_vol.p, s);
  e->flag.alloc(1);
  const FailFlag clear{~0ull};
  FH_CUDA(cudaMemcpyAsync(e->flag.p, &clear, sizeof(clear), cudaMemcpyHostToDevice, s));
  e->stage.alloc(e->V);
  if (e->assembly == FH_ASSEMBLY_EXACT) {
    setup_exact(e.get(), *bnd);
    setup_resident(e.get(), conn, offs, pos);
  } else if (e->precision == 32) {
    setup_tiled<float>(e.get(), *mesh, *bnd, G.p);
    if (e->assembly == FH_ASSEMBLY_ATOMIC) setup_atomic<float>(e.get(), *mesh, G.p);
  } else {
    setup_tiled<double>(e.get(), *mesh, *bnd, G.p);
    if (e->assembly == FH_ASSEMBLY_ATOMIC) setup_atomic<double>(e.get(), *mesh, G.p);
  }
  if (e->assembly != FH_ASSEMBLY_EXACT) {  // exact-order critical dt still needs these
    e->ex.V = e->V;
    e->ex.E = e->E;
    e->ex.n_tet = e->n_tet;
    e->ex.conn = e->conn.p;
    e->ex.row_abs = e->row_abs.p;
    e->ex.csr_offs = e->csr_offs.p;
    e->ex.csr_pos = e->csr_pos.p;
    e->ex.node_vol = e->node_vol.p;
    e->ex.elem_region = e->elem_region.p;
    e->ex.node_region = e->node_region.p;
    e->ex.kfactor = e->kfactor.p;
    e->ex.mats = e->mats_d;
    std::vector<double> nv(e->V), kbh(e->V);
    std::vector<int32_t> nreg(e->V, 0);
    FH_CUDA(cudaMemcpy(nv.data(), e->node_vol.p, sizeof(double) * e->V, cudaMemcpyDeviceToHost));
    if (e->node_region.p)
      FH_CUDA(cudaMemcpy(nreg.data(), e->node_region.p, sizeof(int32_t) * e->V, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < e->V; ++i) {
      const fh_material &m = opts->materials[nreg[i]];
      kbh[i] = (m.perfusion_rate * m.blood_specific_heat) * nv[i];
    }
    e->kb.upload(kbh, s);
    e->ex.kb = e->kb.p;
    if (!e->robin_nodes.empty()) {
      std::vector<int32_t> rs(e->V, -1);
      for (size_t q = 0; q < e->robin_nodes.size(); ++q) rs[e->robin_nodes[q]] = (int32_t)q;
      e->robin_slot.upload(rs, s);
      e->robin_hA_d.upload(e->robin_hA, s);
      e->ex.robin_slot = e->robin_slot.p;
      e->ex.robin_hA = e->robin_hA_d.p;
    }
  }
  FH_CUDA(cudaStreamSynchronize(s));
  *out = e.release();
  FH_API_END
}

int fh_destroy(fh_engine *e) {
  FH_API_BEGIN
  if (e) {
    cudaSetDevice(e->device);
    cudaStreamSynchronize(e->stream);
    delete e;
  }
  FH_API_END
}

int fh_set_temperature(fh_engine *e, const double *T, int64_t n, int64_t step_index, double time) {
  FH_API_BEGIN
  check_engine(e);
  if (n != e->V) fail(FH_ERR_CONFIG, "temperature field has the wrong length");
  FH_CUDA(cudaMemcpyAsync(e->stage.p, T, sizeof(double) * e->V, cudaMemcpyHostToDevice, e->stream));
  if (e->assembly == FH_ASSEMBLY_EXACT)
    FH_CUDA(cudaMemcpyAsync(e->T.p, e->stage.p, sizeof(double) * e->V, cudaMemcpyDeviceToDevice, e->stream));
  else if (e->precision == 32)
    tiled_set_T<float>(e);
  else
    tiled_set_T<double>(e);
  e->step_index = step_index;
  e->time = time;
  e->io_failed = false;
  FH_CUDA(cudaStreamSynchronize(e->stream));
  FH_API_END
}

int fh_get_temperature(fh_engine *e, double *T, int64_t n) {
  FH_API_BEGIN
  check_engine(e);
  if (n != e->V) fail(FH_ERR_CONFIG, "output has the wrong length");
  current_T_to_stage(e);
  FH_CUDA(cudaMemcpyAsync(T, e->stage.p, sizeof(double) * e->V, cudaMemcpyDeviceToHost, e->stream));
  FH_CUDA(cudaStreamSynchronize(e->stream));
  FH_API_END
}

int fh_get_inflow(fh_engine *e, double *F, int64_t n) {
  FH_API_BEGIN
  check_engine(e);
  if (n != e->V) fail(FH_ERR_CONFIG, "output has the wrong length");
  if (e->assembly == FH_ASSEMBLY_EXACT) {
    FH_CUDA(cudaMemcpyAsync(F, e->F.p, sizeof(double) * e->V, cudaMemcpyDeviceToHost, e->stream));
  } else {
    if (!e->keep_inflow) fail(FH_ERR_CONFIG, "TILED mode keeps the inflow only after fh_keep_inflow(e, 1)");
    auto get = [&](auto &st) {
      using S = std::remove_reference_t<decltype(*st.T[0].p)>;
      k_to_old<S><<<nblk(e->V), kBlk, 0, e->stream>>>(st.F.p, e->new_of_old.p, e->V, e->stage.p);
      FH_CUDA(cudaGetLastError());
    };
    if (e->precision == 32) get(*e->tf); else get(*e->tdd);
    FH_CUDA(cudaMemcpyAsync(F, e->stage.p, sizeof(double) * e->V, cudaMemcpyDeviceToHost, e->stream));
  }
  FH_CUDA(cudaStreamSynchronize(e->stream));
  FH_API_END
}

int fh_keep_inflow(fh_engine *e, int32_t on) {
  FH_API_BEGIN
  check_engine(e);
  if (e->assembly == FH_ASSEMBLY_EXACT) return FH_OK;  // EXACT always keeps F
  e->keep_inflow = on != 0;
  if (e->keep_inflow) {
    auto alloc = [&](auto &st) {
      if (!st.F.p) {
        st.F.alloc(e->Vt);
        st.F.zero(e->stream);  // Dirichlet nodes are not updated: their entries stay 0
        FH_CUDA(cudaStreamSynchronize(e->stream));
      }
    };
    if (e->precision == 32) alloc(*e->tf); else alloc(*e->tdd);
  }
  FH_API_END
}

int fh_reset_properties(fh_engine *e) {
  FH_API_BEGIN
  check_engine(e);
  e->frozen = false;
  e->qr_valid = false;
  if (e->assembly != FH_ASSEMBLY_EXACT && !e->td) {  // restore the factor pointers
    if (e->precision == 32) {
      e->tf->args.tet_kf = e->tf->tet_kf.p;
      e->tf->args.hex_kf = e->tf->hex_kf.p;
    } else {
      e->tdd->args.tet_kf = e->tdd->tet_kf.p;
      e->tdd->args.hex_kf = e->tdd->hex_kf.p;
    }
  }
  FH_API_END
}

int fh_step(fh_engine *e, int64_t nsteps, double dt, fh_report *rep) {
  FH_API_BEGIN
  check_engine(e);
  return do_step(e, nsteps, dt, rep);
  FH_API_END
}

int fh_step_timed(fh_engine *e, int64_t nsteps, double dt, fh_report *rep, float *elapsed_ms) {
  FH_API_BEGIN
  check_engine(e);
  return do_step(e, nsteps, dt, rep, elapsed_ms);
  FH_API_END
}

int fh_step_timed_flush(fh_engine *e, int64_t nsteps, double dt, void *scratch, size_t scratch_bytes,
                        fh_report *rep, float *elapsed_ms) {
  FH_API_BEGIN
  check_engine(e);
  if (!scratch || !scratch_bytes) fail(FH_ERR_CONFIG, "scratch buffer required");
  return do_step(e, nsteps, dt, rep, elapsed_ms, scratch, scratch_bytes);
  FH_API_END
}

int fh_step_host_async(fh_engine *e, const double *T_in, double *T_out, int64_t n, int64_t nsteps, double dt,
                       int32_t slot) {
  FH_API_BEGIN
  check_engine(e);
  if (n != e->V) fail(FH_ERR_CONFIG, "field has the wrong length");
  if (slot < 0 || slot > 1) fail(FH_ERR_CONFIG, "slot must be 0 or 1");
  if (e->comm) fail(FH_ERR_CONFIG, "fh_step_host_async is single-GPU only");
  if (nsteps < 0) fail(FH_ERR_CONFIG, "nsteps must be >= 0");
  if (!(dt > 0.0) || !std::isfinite(dt)) fail(FH_ERR_CONFIG, "dt must be positive and finite");
  if (e->io_used[slot]) fail(FH_ERR_CONFIG, "slot still in flight: call fh_host_wait first");
  if (e->io_failed) fail(FH_ERR_CONFIG, "an asynchronous step failed: call fh_set_temperature first");
  e->io_dt = dt;
  if (!e->io_h2d) {
    FH_CUDA(cudaStreamCreateWithFlags(&e->io_h2d, cudaStreamNonBlocking));
    FH_CUDA(cudaStreamCreateWithFlags(&e->io_d2h, cudaStreamNonBlocking));
    for (auto &evs : e->io_ev)
      for (cudaEvent_t &ev : evs) FH_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    FH_CUDA(cudaMallocHost(reinterpret_cast<void **>(&e->io_flag), 2 * sizeof(FailFlag)));
  }
  cudaEvent_t *ev = e->io_ev[slot];
  if (!e->io_in[0].p) {  // both slots at once: no allocation once the pipeline runs
    for (int q = 0; q < 2; ++q) {
      e->io_in[q].alloc(e->V);
      e->io_out[q].alloc(e->V);
      for (int k = 0; k < 4; ++k) FH_CUDA(cudaEventRecord(e->io_ev[q][k], e->stream));  // all free
    }
  }
  // upload on its own stream once the slot's previous field was consumed
  FH_CUDA(cudaStreamWaitEvent(e->io_h2d, ev[1], 0));
  FH_CUDA(cudaMemcpyAsync(e->io_in[slot].p, T_in, sizeof(double) * e->V, cudaMemcpyHostToDevice, e->io_h2d));
  FH_CUDA(cudaEventRecord(ev[0], e->io_h2d));
  // compute stream: field in, steps, field out (into the slot's output buffer
  // once its previous download finished)
  FH_CUDA(cudaStreamWaitEvent(e->stream, ev[0], 0));
  if (e->assembly == FH_ASSEMBLY_EXACT)
    FH_CUDA(cudaMemcpyAsync(e->T.p, e->io_in[slot].p, sizeof(double) * e->V, cudaMemcpyDeviceToDevice, e->stream));
  else if (e->precision == 32)
    tiled_set_T<float>(e, e->io_in[slot].p);
  else
    tiled_set_T<double>(e, e->io_in[slot].p);
  FH_CUDA(cudaEventRecord(ev[1], e->stream));
  {
    // an asynchronous call cannot replay a runaway: several steps per call keep
    // the resident kernel's grid barrier, which stops every CTA at the failing step
    unsigned long long *ll[2] = {e->res.ll[0], e->res.ll[1]};
    if (nsteps > 1) e->res.ll[0] = e->res.ll[1] = nullptr;
    run_steps(e, nsteps, dt);
    e->res.ll[0] = ll[0];
    e->res.ll[1] = ll[1];
  }
  FH_CUDA(cudaMemcpyAsync(&e->io_flag[slot], e->flag.p, sizeof(FailFlag), cudaMemcpyDeviceToHost, e->stream));
  FH_CUDA(cudaStreamWaitEvent(e->stream, ev[3], 0));
  current_T_to_stage(e, e->io_out[slot].p);
  FH_CUDA(cudaEventRecord(ev[2], e->stream));
  // download on its own stream: overlaps the next call's upload and steps
  FH_CUDA(cudaStreamWaitEvent(e->io_d2h, ev[2], 0));
  FH_CUDA(cudaMemcpyAsync(T_out, e->io_out[slot].p, sizeof(double) * e->V, cudaMemcpyDeviceToHost, e->io_d2h));
  FH_CUDA(cudaEventRecord(ev[3], e->io_d2h));
  e->io_used[slot] = true;
  FH_API_END
}

int fh_host_wait(fh_engine *e, int32_t slot, fh_report *rep) {
  FH_API_BEGIN
  check_engine(e);
  if (slot < 0 || slot > 1 || !e->io_used[slot]) fail(FH_ERR_CONFIG, "slot is not in flight");
  FH_CUDA(cudaEventSynchronize(e->io_ev[slot][3]));  // ordered after the flag copy
  e->io_used[slot] = false;
  const FailFlag f = e->io_flag[slot];
  if (rep) {
    std::memset(rep, 0, sizeof(*rep));
    rep->fail_step = -1;
    rep->fail_node = -1;
    rep->time = e->time;
    rep->step_index = e->step_index;
  }
  if (f.step != ~0ull) {
    // the engine stops here: later queued steps were no-ops; the clock goes
    // back to the failing step, the flag is cleared and further async calls
    // are refused until a field is set again (fh_set_temperature)
    FH_CUDA(cudaStreamSynchronize(e->stream));
    const FailFlag clear{~0ull};
    FH_CUDA(cudaMemcpyAsync(e->flag.p, &clear, sizeof(clear), cudaMemcpyHostToDevice, e->stream));
    FH_CUDA(cudaStreamSynchronize(e->stream));
    e->step_index = (int64_t)f.step;
    e->time = (double)f.step * e->io_dt;
    e->io_failed = true;
    if (rep) {
      rep->fail_step = (int64_t)f.step;
      rep->time = e->time;
      rep->step_index = e->step_index;
    }
    fail(FH_ERR_INSTABILITY, "step " + std::to_string((int64_t)f.step) +
                                 ": non-finite or runaway temperature (fh_step_host_async)");
  }
  FH_API_END
}

int fh_step_host(fh_engine *e, const double *T_in, double *T_out, int64_t n, int64_t nsteps, double dt,
                 fh_report *rep) {
  FH_API_BEGIN
  check_engine(e);
  if (n != e->V) fail(FH_ERR_CONFIG, "field has the wrong length");
  if (T_in) {
    FH_CUDA(cudaMemcpyAsync(e->stage.p, T_in, sizeof(double) * e->V, cudaMemcpyHostToDevice, e->stream));
    if (e->assembly == FH_ASSEMBLY_EXACT)
      FH_CUDA(cudaMemcpyAsync(e->T.p, e->stage.p, sizeof(double) * e->V, cudaMemcpyDeviceToDevice, e->stream));
    else if (e->precision == 32)
      tiled_set_T<float>(e);
    else
      tiled_set_T<double>(e);
  }
  const int rc = do_step(e, nsteps, dt, rep);
  if (T_out) {
    current_T_to_stage(e);
    FH_CUDA(cudaMemcpyAsync(T_out, e->stage.p, sizeof(double) * e->V, cudaMemcpyDeviceToHost, e->stream));
    FH_CUDA(cudaStreamSynchronize(e->stream));
  }
  return rc;
  FH_API_END
}

int fh_set_q_static(fh_engine *e, const double *q, int64_t n) {
  FH_API_BEGIN
  check_engine(e);
  if (n != e->V) fail(FH_ERR_CONFIG, "q_static has the wrong length");
  e->q_static.assign(q, q + n);
  if (e->assembly == FH_ASSEMBLY_EXACT) {
    e->qstat.upload(e->q_static, e->stream);
    e->ex.q_static = e->qstat.p;
  } else {
    auto set = [&](auto &st) {
      using S = std::remove_reference_t<decltype(*st.T[0].p)>;
      if (!st.q_ext.p) {
        st.q_ext.alloc(e->Vt);
        st.args.q_ext = st.q_ext.p;
      }
      if (e->load_power.empty()) {
        FH_CUDA(cudaMemcpyAsync(e->stage.p, q, sizeof(double) * n, cudaMemcpyHostToDevice, e->stream));
        float *qf = nullptr;
        double *qd = nullptr;
        if constexpr (sizeof(S) == 4) qf = st.q_ext.p; else qd = st.q_ext.p;
        k_to_new<<<nblk(e->Vt), kBlk, 0, e->stream>>>(e->stage.p, e->old_of_new.p, e->Vt, qf, qd, nullptr, nullptr);
        FH_CUDA(cudaGetLastError());
      } else {
        e->qr_valid = false;  // loads + static power are recombined at the next step
      }
    };
    if (e->precision == 32) set(*e->tf); else set(*e->tdd);
  }
  FH_CUDA(cudaStreamSynchronize(e->stream));
  FH_API_END
}

int fh_set_sources(fh_engine *e, const fh_source *sources, int32_t n) {
  FH_API_BEGIN
  check_engine(e);
  if (n < 0 || n > kMaxSources) fail(FH_ERR_CONFIG, "too many sources");
  e->sources.assign(sources, sources + n);
  if (e->assembly == FH_ASSEMBLY_EXACT) {
    e->ex.n_src = n;
    for (int k = 0; k < n; ++k) e->ex.src[k] = sources[k];
  } else {
    auto setup = [&](auto &st) {
      using S = std::remove_reference_t<decltype(*st.T[0].p)>;
      if (n > 0 && !st.xyz.p) {
        st.xyz.alloc(4 * e->Vt);
        k_xyzv_to_new<S><<<nblk(e->Vt), kBlk, 0, e->stream>>>(e->xyz.p, e->old_of_new.p, st.vol.p, e->Vt, st.xyz.p);
        FH_CUDA(cudaGetLastError());
        st.args.xyzv = st.xyz.p;
      }
    };
    if (e->precision == 32) setup(*e->tf); else setup(*e->tdd);
    FH_CUDA(cudaStreamSynchronize(e->stream));
  }
  FH_API_END
}

int fh_set_probes(fh_engine *e, const int64_t *nodes, int64_t n, int64_t interval, int64_t capacity) {
  FH_API_BEGIN
  check_engine(e);
  if (interval < 1) fail(FH_ERR_CONFIG, "probe interval must be >= 1");
  std::vector<int32_t> p(n);
  for (int64_t q = 0; q < n; ++q) {
    if (nodes[q] < 0 || nodes[q] >= e->V) fail(FH_ERR_CONFIG, "probe node index out of range");
    // TILED multi-GPU: -1 for a node outside this rank's view (recorded as NaN)
    p[q] = (int32_t)(e->assembly == FH_ASSEMBLY_EXACT ? nodes[q] : e->part.new_of_old[nodes[q]]);
  }
  e->probes.upload(p, e->stream);
  e->n_probes = n;
  e->probe_interval = interval;
  e->probe_cap = n ? capacity : 0;
  e->probe_hist.alloc((size_t)std::max<int64_t>(1, n * e->probe_cap));
  e->n_rec = 0;
  e->probe_steps.clear();
  FH_CUDA(cudaStreamSynchronize(e->stream));
  FH_API_END
}

int fh_get_probes(fh_engine *e, double *values, int64_t max_records, int64_t *n_records) {
  FH_API_BEGIN
  check_engine(e);
  const int64_t r = std::min(max_records, e->n_rec);
  if (r > 0)
    FH_CUDA(cudaMemcpyAsync(values, e->probe_hist.p, sizeof(double) * r * e->n_probes, cudaMemcpyDeviceToHost,
                            e->stream));
  FH_CUDA(cudaStreamSynchronize(e->stream));
  *n_records = r;
  FH_API_END
}

int fh_critical_dt(fh_engine *e, const double *T, int64_t n, double *out) {
  FH_API_BEGIN
  check_engine(e);
  if (T && n != e->V) fail(FH_ERR_CONFIG, "field has the wrong length");
  if (!T && e->assembly != FH_ASSEMBLY_EXACT && e->X.world > 1)
    fail(FH_ERR_CONFIG, "a multi-GPU engine holds only its share of the field: pass the gathered field "
                        "(dist.gather_temperature) to fh_critical_dt");
  if (T)
    FH_CUDA(cudaMemcpyAsync(e->stage.p, T, sizeof(double) * e->V, cudaMemcpyHostToDevice, e->stream));
  else
    current_T_to_stage(e);
  e->crit_kbar.alloc(e->E);
  e->crit_lam.alloc(e->V);
  exact_critical(e->ex, e->stage.p, e->crit_kbar.p, e->crit_lam.p, e->stream);
  std::vector<double> lam(e->V);
  FH_CUDA(cudaMemcpyAsync(lam.data(), e->crit_lam.p, sizeof(double) * e->V, cudaMemcpyDeviceToHost, e->stream));
  FH_CUDA(cudaStreamSynchronize(e->stream));
  e->crit_kbar.release();
  e->crit_lam.release();
  double best = -INFINITY;
  bool any = false, nan = false;
  for (double v : lam) {
    if (v == -INFINITY) continue;
    any = true;
    if (std::isnan(v)) nan = true;
    best = std::max(best, v);
  }
  if (!any) fail(FH_ERR_CONFIG, "every node has zero heat capacity");
  if (nan) best = NAN;
  *out = (best <= 0.0) ? INFINITY : 2.0 / best;
  FH_API_END
}

int fh_scatter_loads(fh_engine *e, const double *kbar, const double *T, int64_t n, double *out) {
  FH_API_BEGIN
  check_engine(e);
  if (e->assembly != FH_ASSEMBLY_EXACT) fail(FH_ERR_CONFIG, "scatter_loads needs EXACT mode");
  if (n != e->V) fail(FH_ERR_CONFIG, "field has the wrong length");
  DBuf<double> kb, Tt, o;
  kb.upload(kbar, e->E, e->stream);
  Tt.upload(T, e->V, e->stream);
  o.alloc(e->V);
  exact_scatter(e->ex, kb.p, Tt.p, o.p, e->stream);
  FH_CUDA(cudaMemcpyAsync(out, o.p, sizeof(double) * e->V, cudaMemcpyDeviceToHost, e->stream));
  FH_CUDA(cudaStreamSynchronize(e->stream));
  FH_API_END
}

int fh_get_precompute(fh_engine *e, double *node_volumes, double *elem_volumes) {
  FH_API_BEGIN
  check_engine(e);
  if (node_volumes)
    FH_CUDA(cudaMemcpy(node_volumes, e->node_vol.p, sizeof(double) * e->V, cudaMemcpyDeviceToHost));
  if (elem_volumes)
    FH_CUDA(cudaMemcpy(elem_volumes, e->elem_vol.p, sizeof(double) * e->E, cudaMemcpyDeviceToHost));
  FH_API_END
}

int fh_get_layout(fh_engine *e, fh_layout *out) {
  FH_API_BEGIN
  check_engine(e);
  std::memset(out, 0, sizeof(*out));
  out->n_elements = e->E;
  const int64_t s = e->precision == 32 ? 4 : 8;
  // SURVEY 8(d) canonical: per element N*4 (int32 conn) + 6s (G) + 4 (factor, if any);
  // per node 2s (T r/w) + s (v) + per-node source data
  int64_t canon = e->n_tet * (16 + 6 * s) + e->n_hex * (32 + 6 * s) + (e->kfactor.p ? 4 * e->E : 0);
  canon += e->V * 3 * s;
  if (!e->q_static.empty() || !e->load_power.empty()) canon += e->V * s;
  if (!e->sources.empty()) canon += e->V * 3 * s;
  out->canonical_bytes = canon;
  if (e->assembly == FH_ASSEMBLY_EXACT) {
    out->kernels_per_step = e->resident ? 0 : 2;
    out->resident_ctas = e->resident ? e->res_ctas : 0;
    out->resident_threads = e->resident ? e->res_threads : 0;
    out->n_slots = e->E;
    out->n_nodes_owned = e->V;
    // conn + A + contrib w/r + csr + node streams
    out->step_bytes = e->nconn * 4 + (16 * e->n_tet + 64 * e->n_hex) * 8 + e->nconn * 16 + e->nconn * 4 +
                      e->V * 8 * 8;
  } else {
    const Partition &P = e->part;
    auto launches = [&](const auto &st) {  // one per tile kind present in each launch range
      const int ni = st.n_parts_local - st.n_boundary;
      return (st.n_mixed_i > 0 && st.n_mixed_i < ni ? 2 : 1) + (st.n_lean_i > 0 && st.n_lean_i < ni - st.n_mixed_i ? 1 : 0) +
             (st.n_mixed_i < ni && st.n_lean_mixed_i > 0 && st.n_lean_mixed_i < st.n_mixed_i ? 1 : 0) +
             (st.n_boundary ? (st.n_mixed_b > 0 && st.n_mixed_b < st.n_boundary ? 2 : 1) : 0);
    };
    out->kernels_per_step = e->precision == 32 ? launches(*e->tf) : launches(*e->tdd);
    if (e->assembly == FH_ASSEMBLY_ATOMIC) out->kernels_per_step = (e->n_tet ? 1 : 0) + (e->n_hex ? 1 : 0) + 1;
    out->n_parts = P.n_parts;
    out->max_part_nodes = P.max_part_nodes;
    const int64_t nts = (int64_t)P.tet_slot_elem.size(), nhs = (int64_t)P.hex_slot_elem.size();
    out->n_slots = nts + nhs;
    int64_t owned = 0;
    for (int p = 0; p < P.n_parts; ++p) owned += P.part_n_free[p];
    out->n_nodes_owned = owned;
    // slot streams as stored: 16-bit connectivity, G (conductivity factor
    // folded in when temperature-dependent), frozen kbar (TI), material byte,
    // per-corner rank (ranked mode) or per-slot phase (colour mode)
    const bool regions = (e->tf && e->tf->hex_region.p) || (e->tf && e->tf->tet_region.p) ||
                         (e->tdd && e->tdd->hex_region.p) || (e->tdd && e->tdd->tet_region.p);
    const int hex_mode = e->tf ? e->tf->mode : (e->tdd ? e->tdd->mode : 0);
    int64_t b = nts * (8 + 6 * s) + nhs * (16 + 6 * s);
    if (!e->td) b += (nts + nhs) * s;
    if (regions) b += nts + nhs;
    if (P.colored_ok) b += nts; else b += nts * 4;
    if (hex_mode == kModeRanked) b += nhs * 8;
    if (hex_mode == kModeColored) b += nhs;
    int64_t node_streams = 3 * s;  // T read, T' write, v
    if (!e->td) node_streams += s;  // frozen capacity
    if (!e->q_static.empty() || !e->load_power.empty()) node_streams += s;
    if (!e->sources.empty()) node_streams += 3 * s;
    b += owned * node_streams;
    b += (int64_t)P.halo_nodes.size() * s;  // halo temperatures (each tile stages its own)
    out->step_bytes = b;
  }
  FH_API_END
}

void *fh_stream(fh_engine *e) { return e ? (void *)e->stream : nullptr; }

int fh_get_node_order(fh_engine *e, int64_t *new_to_old, int64_t n) {
  FH_API_BEGIN
  check_engine(e);
  if (n != e->V) fail(FH_ERR_CONFIG, "output has the wrong length");
  if (e->assembly == FH_ASSEMBLY_EXACT) {
    for (int64_t i = 0; i < n; ++i) new_to_old[i] = i;
  } else {  // multi-GPU: the rank's local order (owned, then halo nodes), then -1
    const int64_t nl = (int64_t)e->part.old_of_new.size();
    std::memcpy(new_to_old, e->part.old_of_new.data(), sizeof(int64_t) * nl);
    for (int64_t i = nl; i < n; ++i) new_to_old[i] = -1;
  }
  FH_API_END
}

// ---------------------------------------------------------------------------
// operator layer
static Curve<double> make_curve(const double *x, const double *y, int64_t n) {
  fh_curve c{(int32_t)n, x, y};
  Curve<double> out;
  fill_curve(out, c, "curve");
  return out;
}

int fh_eval_curve_nodes(const double *xs, const double *ys, int64_t n_knots, const double *temps, int64_t n,
                        double *out) {
  FH_API_BEGIN
  const Curve<double> c = make_curve(xs, ys, n_knots);
  DBuf<double> T, o;
  T.upload(temps, n);
  o.alloc(n);
  op_curve(c, T.p, n, o.p, 0);
  FH_CUDA(cudaMemcpy(out, o.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
  FH_API_END
}

int fh_lumped_capacity_nodes(const double *rho_x, const double *rho_y, int64_t n_rho, const double *c_x,
                             const double *c_y, int64_t n_c, const double *temps, const double *vols, int64_t n,
                             double *out) {
  FH_API_BEGIN
  const Curve<double> r = make_curve(rho_x, rho_y, n_rho), c = make_curve(c_x, c_y, n_c);
  DBuf<double> T, v, o;
  T.upload(temps, n);
  v.upload(vols, n);
  o.alloc(n);
  op_capacity(r, c, T.p, v.p, n, o.p, 0);
  FH_CUDA(cudaMemcpy(out, o.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
  FH_API_END
}

int fh_element_mean_nodal(const int64_t *conn_data, const int64_t *conn_offs, int64_t n_elem, const double *nodal,
                          int64_t n_nodes, double *out) {
  FH_API_BEGIN
  const int64_t nc = conn_offs[n_elem];
  std::vector<int32_t> c32(nc);
  for (int64_t p = 0; p < nc; ++p) {
    if (conn_data[p] < 0 || conn_data[p] >= n_nodes) fail(FH_ERR_CONFIG, "node index out of range");
    c32[p] = (int32_t)conn_data[p];
  }
  DBuf<int32_t> c;
  DBuf<int64_t> offs;
  DBuf<double> nd, o;
  c.upload(c32);
  offs.upload(conn_offs, n_elem + 1);
  nd.upload(nodal, n_nodes);
  o.alloc(n_elem);
  op_mean(c.p, offs.p, n_elem, nd.p, o.p, 0);
  FH_CUDA(cudaMemcpy(out, o.p, sizeof(double) * n_elem, cudaMemcpyDeviceToHost));
  FH_API_END
}

int fh_scatter_net_loads(const int64_t *conn_data, const int64_t *conn_offs, const double *mat_data,
                         const int64_t *mat_offs, int64_t n_elem, const double *kbar, const double *temps,
                         int64_t n_nodes, int64_t chunk_size, double *out) {
  FH_API_BEGIN
  if (chunk_size < 1) fail(FH_ERR_CONFIG, "chunk_size must be >= 1");
  const int64_t nc = conn_offs[n_elem];
  std::vector<int32_t> c32(nc), elem_of(nc);
  for (int64_t e = 0; e < n_elem; ++e) {
    const int64_t n = conn_offs[e + 1] - conn_offs[e];
    if (n < 1 || n > 8) fail(FH_ERR_CONFIG, "elements must have 1..8 nodes");
    if (mat_offs[e + 1] - mat_offs[e] != n * n) fail(FH_ERR_CONFIG, "mat_offs do not match conn_offs");
    for (int64_t p = conn_offs[e]; p < conn_offs[e + 1]; ++p) elem_of[p] = (int32_t)e;
  }
  std::vector<int32_t> offs(n_nodes + 1, 0), pos(nc);
  for (int64_t p = 0; p < nc; ++p) {
    if (conn_data[p] < 0 || conn_data[p] >= n_nodes) fail(FH_ERR_CONFIG, "node index out of range");
    c32[p] = (int32_t)conn_data[p];
    offs[c32[p] + 1]++;
  }
  for (int64_t i = 0; i < n_nodes; ++i) offs[i + 1] += offs[i];
  std::vector<int32_t> fill(offs.begin(), offs.end() - 1);
  for (int64_t p = 0; p < nc; ++p) pos[fill[c32[p]]++] = (int32_t)p;
  DBuf<int32_t> dc, deo, doffs, dpos;
  DBuf<int64_t> dco, dmo;
  DBuf<double> dm, dk, dT, dcontrib, dout;
  dc.upload(c32);
  deo.upload(elem_of);
  doffs.upload(offs);
  dpos.upload(pos);
  dco.upload(conn_offs, n_elem + 1);
  dmo.upload(mat_offs, n_elem + 1);
  dm.upload(mat_data, mat_offs[n_elem]);
  dk.upload(kbar, n_elem);
  dT.upload(temps, n_nodes);
  dcontrib.alloc(nc);
  dout.alloc(n_nodes);
  ExactArgs g;
  std::memset(&g, 0, sizeof(g));
  g.V = n_nodes;
  g.E = n_elem;
  g.chunk_size = chunk_size;
  g.conn = dc.p;
  g.conn_offs = dco.p;
  g.mat_offs = dmo.p;
  g.mat = dm.p;
  g.csr_offs = doffs.p;
  g.csr_pos = dpos.p;
  g.elem_of = deo.p;
  g.contrib = dcontrib.p;
  exact_scatter(g, dk.p, dT.p, dout.p, 0);
  FH_CUDA(cudaMemcpy(out, dout.p, sizeof(double) * n_nodes, cudaMemcpyDeviceToHost));
  FH_API_END
}

int fh_nodal_update(double *temps, const double *inflow, const double *capacity, const double *perf_k,
                    const double *perf_q, const double *metab_q, const double *extra_q, int64_t n, double dt) {
  FH_API_BEGIN
  DBuf<double> T, F, C, kb, qb, qm, qr;
  T.upload(temps, n);
  F.upload(inflow, n);
  C.upload(capacity, n);
  kb.upload(perf_k, n);
  qb.upload(perf_q, n);
  qm.upload(metab_q, n);
  qr.upload(extra_q, n);
  op_update(T.p, F.p, C.p, kb.p, qb.p, qm.p, qr.p, n, dt, 0);
  FH_CUDA(cudaMemcpy(temps, T.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
  FH_API_END
}

int fh_nccl_library(const char *path) {
  FH_API_BEGIN
  nccl_set_library(path);
  FH_API_END
}

int fh_nccl_unique_id(char *id128) {
  FH_API_BEGIN
  NcclUniqueId id;
  nccl_unique_id(&id);
  std::memcpy(id128, id.internal, sizeof(id.internal));
  FH_API_END
}

int fh_attach_transport(fh_engine *e, const fh_transport *t) {
  FH_API_BEGIN
  check_engine(e);
  if (e->assembly != FH_ASSEMBLY_TILED) fail(FH_ERR_CONFIG, "multi-GPU needs TILED mode");
  if (!t || !t->exchange || !t->allreduce_min_u64) fail(FH_ERR_CONFIG, "transport needs both callbacks");
  if (e->comm) fail(FH_ERR_CONFIG, "the engine already uses NCCL");
  e->transport = *t;
  FH_API_END
}

int fh_attach_nccl(fh_engine *e, const char *id128, int32_t rank, int32_t world) {
  FH_API_BEGIN
  check_engine(e);
  if (e->assembly != FH_ASSEMBLY_TILED) fail(FH_ERR_CONFIG, "multi-GPU needs TILED mode");
  if (world != e->X.world || rank != e->X.rank)
    fail(FH_ERR_CONFIG, "rank/world do not match the engine's domain range");
  if (!e->comm) {  // world 1: a one-rank communicator (only the fail-flag all-reduce uses it)
    NcclUniqueId id;
    std::memcpy(id.internal, id128, sizeof(id.internal));
    e->comm = nccl_comm_init(id, rank, world);
  }
  FH_API_END
}

// halo bookkeeping of the engine (original node ids) and a host-side exchange
// used when ranks share one GPU in tests (no kernels wait on one another)
int fh_halo_info(fh_engine *e, int32_t *world, int32_t *rank, int32_t *n_peers, int64_t *n_send, int64_t *n_recv,
                 int64_t *n_boundary_parts, int64_t *n_parts) {
  FH_API_BEGIN
  check_engine(e);
  *world = e->X.world;
  *rank = e->X.rank;
  *n_peers = (int32_t)e->X.peers.size();
  *n_send = (int64_t)e->X.send_nodes.size();
  *n_recv = (int64_t)e->X.recv_nodes.size();
  *n_boundary_parts = e->X.n_boundary;
  *n_parts = (int64_t)e->X.part_order.size();
  FH_API_END
}

int fh_halo_lists(fh_engine *e, int32_t *peers, int64_t *send_offs, int64_t *send_nodes, int64_t *recv_offs,
                  int64_t *recv_nodes) {
  FH_API_BEGIN
  check_engine(e);
  const Exchange &X = e->X;
  for (size_t q = 0; q < X.peers.size(); ++q) peers[q] = X.peers[q];
  for (size_t q = 0; q < X.send_offs.size(); ++q) send_offs[q] = X.send_offs[q];
  for (size_t q = 0; q < X.recv_offs.size(); ++q) recv_offs[q] = X.recv_offs[q];
  for (size_t q = 0; q < X.send_nodes.size(); ++q) send_nodes[q] = e->part.old_of_new[X.send_nodes[q]];
  for (size_t q = 0; q < X.recv_nodes.size(); ++q) recv_nodes[q] = e->part.old_of_new[X.recv_nodes[q]];
  FH_API_END
}

}  // extern "C"

template <typename S>
static void halo_host_io(fh_engine *e, double *out, const double *in) {
  TiledState<S> &st = tstate<S>(e);
  const bool exp = out != nullptr;
  const std::vector<int32_t> &nodes = exp ? e->X.send_nodes : e->X.recv_nodes;
  const int64_t n = (int64_t)nodes.size();
  if (!n) return;
  std::vector<S> h(n);
  DBuf<S> buf;
  buf.alloc(n);
  const int32_t *idx = exp ? e->x_send.p : e->x_recv.p;
  if (exp) {
    halo_pack<S>(st.T[st.cur].p, idx, n, buf.p, e->stream);
    FH_CUDA(cudaMemcpyAsync(h.data(), buf.p, sizeof(S) * n, cudaMemcpyDeviceToHost, e->stream));
    FH_CUDA(cudaStreamSynchronize(e->stream));
    for (int64_t q = 0; q < n; ++q) out[q] = (double)h[q];
  } else {
    for (int64_t q = 0; q < n; ++q) h[q] = (S)in[q];
    FH_CUDA(cudaMemcpyAsync(buf.p, h.data(), sizeof(S) * n, cudaMemcpyHostToDevice, e->stream));
    halo_unpack<S>(st.T[st.cur].p, idx, n, buf.p, e->stream);
    FH_CUDA(cudaStreamSynchronize(e->stream));
  }
}

extern "C" {

int fh_halo_export(fh_engine *e, double *send_values) {
  FH_API_BEGIN
  check_engine(e);
  if (e->X.world < 2) fail(FH_ERR_CONFIG, "engine has no halo");
  if (e->precision == 32) halo_host_io<float>(e, send_values, nullptr); else halo_host_io<double>(e, send_values, nullptr);
  FH_API_END
}

int fh_halo_import(fh_engine *e, const double *recv_values) {
  FH_API_BEGIN
  check_engine(e);
  if (e->X.world < 2) fail(FH_ERR_CONFIG, "engine has no halo");
  if (e->precision == 32) halo_host_io<float>(e, nullptr, recv_values); else halo_host_io<double>(e, nullptr, recv_values);
  FH_API_END
}

// owned-node mask in the original numbering (1 = this engine updates / owns it)
int fh_get_owned(fh_engine *e, uint8_t *mask, int64_t n) {
  FH_API_BEGIN
  check_engine(e);
  if (n != e->V) fail(FH_ERR_CONFIG, "output has the wrong length");
  if (e->assembly == FH_ASSEMBLY_EXACT) {
    std::memset(mask, 1, (size_t)n);
  } else {
    std::memset(mask, 0, (size_t)n);
    for (int64_t v = e->X.node_lo; v < e->X.node_hi; ++v) mask[e->part.old_of_new[v]] = 1;
  }
  FH_API_END
}

// ---------------------------------------------------------------------------
// host-only partition plan (no GPU): the bookkeeping of fh_create for a rank
struct fh_plan {
  Partition P;
  Exchange X;
  // the rank's local view (localize_partition): what its engine keeps on the device
  int64_t rank_slots = 0, rank_real_slots = 0, rank_local_nodes = 0, rank_owned_nodes = 0, rank_step_bytes = 0,
          rank_device_bytes = 0;
};

int fh_plan_create(const fh_mesh *mesh, const fh_boundary *bnd, const fh_options *opts, int32_t world, int32_t rank,
                   fh_plan **out) {
  FH_API_BEGIN
  auto pl = std::make_unique<fh_plan>();
  const int64_t V = mesh->n_nodes;
  std::vector<uint8_t> cls(V, 0);
  for (int64_t q = 0; q < bnd->n_robin; ++q) cls[bnd->robin_nodes[q]] = 1;
  for (int64_t q = 0; q < bnd->n_dirichlet; ++q) cls[bnd->dirichlet_nodes[q]] = 2;
  PartitionInput pin{};
  pin.V = V;
  pin.n_tet = mesh->n_tets;
  pin.n_hex = mesh->n_hexes;
  pin.xyz = mesh->coords;
  pin.tets = mesh->tets;
  pin.hexes = mesh->hexes;
  pin.node_class = cls.data();
  pin.target_part_nodes = opts->part_nodes > 0 ? opts->part_nodes : default_part_nodes(opts->precision, mesh->n_tets, mesh->n_hexes);
  // the engine's default tile size, first pass (the second, occupancy-measured
  // pass needs a GPU: pass part_nodes explicitly to pin the plan)
  if (opts->part_nodes <= 0 && mesh->n_nodes / pin.target_part_nodes < 2 * 148)
    pin.target_part_nodes = (int)std::max<int64_t>(96, mesh->n_nodes / (2 * 148));
  else if (opts->part_nodes <= 0)
    pin.target_part_nodes = wave_fit_part_nodes(pin.target_part_nodes, mesh->n_nodes, std::max(1, opts->n_domains),
                                                opts->precision, mesh->n_tets, mesh->n_hexes, opts->device);
  pin.batch = kBatch;
  // layout tuning knobs (fh_options): hex colour order, first-touch node order
  pin.hex_color = opts->hex_color;
  pin.first_touch = opts->first_touch;
  pin.tet_rows = default_tet_rows(mesh->n_tets, mesh->n_hexes, opts->tet_rows, opts->precision);
  pin.n_domains = std::max(1, opts->n_domains);
  pin.slab_axis = opts->slab_axis;
  build_partition(pin, pl->P);
  std::vector<uint8_t> is_dir(V, 0);
  for (int64_t q = 0; q < bnd->n_dirichlet; ++q) is_dir[pl->P.new_of_old[bnd->dirichlet_nodes[q]]] = 1;
  build_exchange(pl->P, is_dir.data(), pin.n_domains, world, rank, pl->X);
  {
    Exchange Xc = pl->X;
    Partition L;
    localize_partition(pl->P, Xc, L);
    const int64_t sb = opts->precision == 32 ? 4 : 8;
    const int64_t nts = (int64_t)L.tet_slot_elem.size(), nhs = (int64_t)L.hex_slot_elem.size();
    int64_t real = 0;
    for (int p = 0; p < L.n_parts; ++p) real += L.part_tet_count[p] + L.part_hex_count[p];
    pl->rank_slots = nts + nhs;
    pl->rank_real_slots = real;
    pl->rank_local_nodes = (int64_t)L.old_of_new.size();
    pl->rank_owned_nodes = Xc.node_hi - Xc.node_lo;
    // per step: slot records (16-bit conn + 6 G) + T read/write and v of the owned nodes + halo T reads
    const int64_t rec = nts * (8 + 6 * sb) + nhs * (16 + 6 * sb);
    pl->rank_step_bytes = rec + pl->rank_owned_nodes * 3 * sb + (pl->rank_local_nodes - pl->rank_owned_nodes) * sb;
    // resident step arrays: records, T[2] and v (local nodes), halo id lists, tile tables
    pl->rank_device_bytes = rec + pl->rank_local_nodes * 3 * sb + 4 * (int64_t)L.halo_nodes.size() +
                            4 * 12 * (int64_t)(L.n_parts + 1);
  }
  *out = pl.release();
  FH_API_END
}

static int64_t sum_u8(const std::vector<uint8_t> &v) {
  int64_t t = 0;
  for (uint8_t x : v) t += x;
  return t;
}

int fh_plan_info(fh_plan *pl, int64_t *info, int32_t n_info) {
  FH_API_BEGIN
  const int64_t v[] = {pl->P.n_parts, pl->X.part_hi - pl->X.part_lo, pl->X.n_boundary, (int64_t)pl->X.peers.size(),
                       (int64_t)pl->X.send_nodes.size(), (int64_t)pl->X.recv_nodes.size(), pl->X.node_lo,
                       pl->X.node_hi, (int64_t)pl->P.corner_unique, pl->P.max_phase_tet, pl->P.max_phase_hex,
                       (int64_t)(pl->P.tet_slot_elem.size() + pl->P.hex_slot_elem.size()), pl->P.max_local_nodes,
                       (int64_t)pl->P.colored_ok, pl->P.max_colors, pl->P.max_nph_tet, pl->P.max_nph_hex,
                       sum_u8(pl->P.tet_batch_nph), (int64_t)pl->P.tet_batch_nph.size(), sum_u8(pl->P.hex_batch_nph),
                       (int64_t)pl->P.hex_batch_nph.size(), pl->rank_slots, pl->rank_real_slots, pl->rank_local_nodes,
                       pl->rank_owned_nodes, pl->rank_step_bytes, pl->rank_device_bytes};
  for (int q = 0; q < n_info && q < (int)(sizeof(v) / sizeof(v[0])); ++q) info[q] = v[q];
  FH_API_END
}

int fh_plan_arrays(fh_plan *pl, int64_t *new_to_old, int64_t *part_node_start, int32_t *peers, int64_t *send_offs,
                   int64_t *send_nodes, int64_t *recv_offs, int64_t *recv_nodes) {
  FH_API_BEGIN
  const Partition &P = pl->P;
  const Exchange &X = pl->X;
  if (new_to_old) std::memcpy(new_to_old, P.old_of_new.data(), sizeof(int64_t) * P.old_of_new.size());
  if (part_node_start)
    for (size_t q = 0; q < P.part_node_start.size(); ++q) part_node_start[q] = P.part_node_start[q];
  if (peers)
    for (size_t q = 0; q < X.peers.size(); ++q) peers[q] = X.peers[q];
  if (send_offs)
    for (size_t q = 0; q < X.send_offs.size(); ++q) send_offs[q] = X.send_offs[q];
  if (recv_offs)
    for (size_t q = 0; q < X.recv_offs.size(); ++q) recv_offs[q] = X.recv_offs[q];
  if (send_nodes)
    for (size_t q = 0; q < X.send_nodes.size(); ++q) send_nodes[q] = P.old_of_new[X.send_nodes[q]];
  if (recv_nodes)
    for (size_t q = 0; q < X.recv_nodes.size(); ++q) recv_nodes[q] = P.old_of_new[X.recv_nodes[q]];
  FH_API_END
}

int fh_plan_destroy(fh_plan *pl) {
  delete pl;
  return FH_OK;
}

}  // extern "C"
