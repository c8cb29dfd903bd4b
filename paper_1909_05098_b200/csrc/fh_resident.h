// Resident small-mesh path of the EXACT step (fh_resident.cu).
#pragma once
#include <vector>

#include "fh_exact_dev.cuh"

namespace fh {

// threads per resident CTA at most (launch bounds: up to 128 registers per thread)
constexpr int kResThreads = 512;

// Host-built layout: the nodes are cut into n_cta contiguous ranges (one CTA
// each, balanced by incidences); every CTA keeps, for the whole launch, the
// A rows of the incidences of its nodes in shared memory and stages the
// temperatures of its nodes plus their halo once per step.
struct ResidentPlan {
  int n_cta = 0;
  int threads = 0;
  int max_local = 0, max_inc = 0, max_own = 0;  // per CTA: owned + halo nodes, incidences, owned nodes
  size_t smem = 0;                               // dynamic shared memory per CTA
  size_t off_K = 0, off_A = 0, off_C = 0, off_Kb = 0, off_L = 0, off_E = 0, off_I = 0, off_H = 0, off_N = 0,
         off_O = 0;
  std::vector<int32_t> cta_node, cta_halo, halo_nodes, cta_inc;  // n_cta + 1 offsets, halo ids
  std::vector<uint16_t> inc_lconn;       // 8 per incidence: tile-local node of each element corner
  std::vector<int32_t> inc_elem;         // element of each incidence
  std::vector<uint8_t> inc_info;         // corner | (8 nodes ? 8 : 0) | (opens a chunk ? 16 : 0)
};

// Builds the plan for `n_cta` CTAs of `threads` threads.  Returns false when
// a CTA's working set does not fit `smem_limit` bytes of shared memory.
bool build_resident_plan(int64_t V, int64_t n_tet, int64_t chunk_size, const std::vector<int32_t> &conn,
                         const std::vector<int32_t> &csr_offs, const std::vector<int32_t> &csr_pos, int n_cta,
                         bool stage_k, bool frozen_kbar_slots, size_t smem_limit, ResidentPlan &plan);

struct ResidentArgs {
  ExactArgs g;
  const int32_t *cta_node, *cta_halo, *halo_nodes, *cta_inc;
  const uint16_t *inc_lconn;
  const int32_t *inc_elem;
  const uint8_t *inc_info;
  uint32_t off_K, off_A, off_C, off_Kb, off_L, off_E, off_I, off_H, off_N, off_O;
  double *T0, *T1;        // T0: the engine's field (in and out), T1: ping-pong scratch
  unsigned long long *bar;  // grid barrier word (stamped mode: set to 1 by a CTA that lost its neighbours), zeroed before every launch
  // stamped mode (null: grid barrier): two buffers of 2 words per node, {value half | stamp << 32};
  // the field at the start of step j of the launch carries stamp0 + j in ll[j & 1]
  unsigned long long *ll[2];
  uint32_t stamp0;
  int64_t step0;          // steps taken before this launch
  int64_t nsteps;
  double time0, dt;       // start time of the first step; later steps start at (step0 + j) * dt
  const int32_t *probes;  // probe nodes, recorded after every step whose index is a multiple of interval
  int64_t n_probes, probe_interval, rec0, rec_cap;
  double *probe_out;
};

// one launch = nsteps steps (cooperative: all CTAs co-resident)
void resident_run(const ResidentArgs &r, int n_cta, int threads, size_t smem, bool td, bool stage_k,
                  cudaStream_t s);
// CTAs of `threads` threads with `smem` bytes that stay resident per SM
int resident_occupancy(bool td, bool stage_k, int threads, size_t smem);

}  // namespace fh
