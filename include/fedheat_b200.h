/*
 * fedheat_b200.h -- C ABI of the B200-native FED-FEM bio-heat engine
 * (libfedheat_b200.so).  Plain pointers and sizes only; no torch or CUDA
 * types cross this boundary.  Host arrays are borrowed for the duration of a
 * call; every device buffer is owned by the library.
 *
 * Two layers, each a drop-in for a layer of the reference package
 * (/root/reference/pkg/src/fedheat/, cited file:line below):
 *
 *  1. Operator layer -- one entry point per numba kernel of kernels.py, same
 *     argument meaning, caller-allocated outputs, bit-identical results.  A
 *     maintainer swaps the numba bodies for these (INTEGRATION.md shows the
 *     ctypes stub).  Each call copies its inputs to the GPU, runs one CUDA
 *     kernel and copies the result back.
 *
 *  2. Engine layer -- the stateful step path of solver.ExplicitEngine
 *     (solver.py:243-519): mesh/material/boundary upload and device
 *     precompute in fh_create, device-resident stepping in fh_step.
 *
 * Status codes: 0 ok, 1 config error (ConfigError), 2 instability
 * (InstabilityError), 3 CUDA/NCCL failure, 4 degenerate element
 * (DegenerateElementError), 5 mesh text format (MeshFormatError).  fh_last_error() returns the calling thread's
 * message for the last non-zero status.
 */
#ifndef FEDHEAT_B200_H
#define FEDHEAT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FH_OK 0
#define FH_ERR_CONFIG 1
#define FH_ERR_INSTABILITY 2
#define FH_ERR_DEVICE 3
#define FH_ERR_DEGENERATE 4
#define FH_ERR_FORMAT 5 /* MeshFormatError (mesh ingest) */

#define FH_MAX_KNOTS 32
#define FH_CHUNK_SIZE 4096 /* solver.py:48 CHUNK_SIZE */

const char *fh_last_error(void);
int fh_version(void);
int fh_device_count(int *count);

/* ------------------------------------------------------------------ */
/* 1. Operator layer (kernels.py:76-142).  All arrays are host memory. */
/* ------------------------------------------------------------------ */

/* kernels.py:76-79 eval_curve_nodes(xs, ys, temps, out) */
int fh_eval_curve_nodes(const double *xs, const double *ys, int64_t n_knots, const double *temps,
                        int64_t n, double *out);

/* kernels.py:82-86 lumped_capacity_nodes(rho_x, rho_y, c_x, c_y, temps, vols, out) */
int fh_lumped_capacity_nodes(const double *rho_x, const double *rho_y, int64_t n_rho, const double *c_x,
                             const double *c_y, int64_t n_c, const double *temps, const double *vols,
                             int64_t n, double *out);

/* kernels.py:89-98 element_mean_nodal(conn_data, conn_offs, nodal, out) */
int fh_element_mean_nodal(const int64_t *conn_data, const int64_t *conn_offs, int64_t n_elem,
                          const double *nodal, int64_t n_nodes, double *out);

/* kernels.py:101-134 scatter_net_loads(conn_data, conn_offs, mat_data, mat_offs, kbar, temps,
 * n_chunks, chunk_size, buffers, out) -- the O(n_chunks * n_nodes) `buffers`
 * scratch of the reference is not needed; the chunk semantics (private
 * partial per chunk_size elements, partials added in chunk order) are kept. */
int fh_scatter_net_loads(const int64_t *conn_data, const int64_t *conn_offs, const double *mat_data,
                         const int64_t *mat_offs, int64_t n_elem, const double *kbar, const double *temps,
                         int64_t n_nodes, int64_t chunk_size, double *out);

/* kernels.py:137-142 nodal_update(temps, inflow, capacity, perf_k, perf_q, metab_q, extra_q, dt);
 * temps is updated in place. */
int fh_nodal_update(double *temps, const double *inflow, const double *capacity, const double *perf_k,
                    const double *perf_q, const double *metab_q, const double *extra_q, int64_t n,
                    double dt);

/* ------------------------------------------------------------------ */
/* 2. Engine layer (solver.py:243-519)                                  */
/* ------------------------------------------------------------------ */

typedef struct fh_engine fh_engine;

typedef struct {
  int32_t n; /* knots, 1..FH_MAX_KNOTS; 0 = absent (only for `perfusion`) */
  const double *x;
  const double *y;
} fh_curve;

/* material.py:65-123 TissueMaterial; `perfusion` (extension) makes the
 * perfusion rate temperature dependent and replaces perfusion_rate. */
typedef struct {
  fh_curve density, specific_heat, conductivity, perfusion;
  double perfusion_rate, blood_specific_heat, arterial_temperature, metabolic_rate;
} fh_material;

/* mesh.py:38-59 Mesh: nodes (V,3) float64, tets (Et,4), hexes (Eh,8) int64;
 * global element order = tets then hexes. */
typedef struct {
  int64_t n_nodes;
  const double *coords;
  int64_t n_tets;
  const int64_t *tets;
  int64_t n_hexes;
  const int64_t *hexes;
} fh_mesh;

#define FH_SOURCE_GAUSSIAN 0 /* amp * exp(-|x - c(t)|^2 / (2 sigma^2)), c(t) = x0 + vel * t */
#define FH_SOURCE_RF 1       /* min(amp / (4 pi |x - x0|^2), cap) */
typedef struct {
  int32_t kind;
  double amp, sigma, cap;
  double x0[3], vel[3];
  double t0, t1; /* active while t0 <= t < t1 (t = step start time) */
} fh_source;

/* solver.py:91-164 BoundarySpec after resolve_boundary, plus extensions. */
typedef struct {
  int64_t n_dirichlet; /* sorted unique node ids, values */
  const int64_t *dirichlet_nodes;
  const double *dirichlet_values;
  int64_t n_loads; /* heat_loads: nodes of load l are load_nodes[load_offsets[l]:load_offsets[l+1]] */
  const int64_t *load_offsets;
  const int64_t *load_nodes;
  const double *load_power, *load_t0, *load_t1;
  const double *q_static; /* extension: (V,) static nodal power in W, or NULL */
  int32_t n_sources;      /* extension: volumetric sources lumped as Q(x_i, t) * v_i */
  const fh_source *sources;
  int64_t n_robin; /* extension: convective nodes, rate += hA*(Tinf) - hA*T */
  const int64_t *robin_nodes;
  const double *robin_hA, *robin_hAT;
} fh_boundary;

#define FH_ASSEMBLY_EXACT 0  /* fp64, reference operation order, bitwise == reference */
#define FH_ASSEMBLY_TILED 1  /* fused owner-computes tiles, G-form, deterministic */
#define FH_ASSEMBLY_ATOMIC 2 /* element kernel + red.global into F, then node update (tolerance only) */

typedef struct {
  int32_t precision; /* 64 or 32 (32 only for TILED / ATOMIC) */
  int32_t assembly;
  int32_t td_mode;   /* 1: refresh properties every step; 0: freeze at first step */
  int32_t device;    /* CUDA ordinal */
  double runaway_limit;
  int32_t n_materials; /* >= 1; >1 = regions (extension) */
  const fh_material *materials;
  const int32_t *element_region;  /* (E,) or NULL */
  const double *element_kfactor;  /* (E,) or NULL: extension, kbar_e *= f_e */
  int32_t part_nodes;             /* TILED: nodes per tile (0 = default) */
  int32_t n_domains;              /* multi-GPU: domains the mesh is cut into (1, 2, 4 or 8) */
  int32_t domain_lo, domain_hi;   /* this engine owns domains [lo, hi) */
  int32_t slab_axis;              /* -1: recursive coordinate bisection; 0/1/2: domains are slabs */
  /* Tuning knobs.  0 selects the measured default everywhere; the values are
   * explicit so that no environment variable changes what the library does. */
  int32_t exact_resident;   /* EXACT: 0 auto (resident many-steps-per-launch kernel when the mesh's
                               per-CTA working set fits shared memory), 1 off (two launches per step),
                               2 required (FH_ERR_CONFIG when it does not fit) */
  int32_t resident_ctas;    /* resident path: CTA count (0: one per SM) */
  int32_t tile_mode;        /* TILED hex accumulation mode + 1 (0: default) */
  int32_t tile_stages;      /* TILED TMA ring depth (0: default 2) */
  int32_t tet_rows;         /* TILED tet accumulator rows: 0 default (4 on tet-only meshes), or 1..4 */
  int32_t launch_order;     /* TILED: 0 default, 1 partition (RCB) order, 2 longest tiles first */
  int32_t kind_split;       /* TILED mixed meshes: 0 default (split hex-only tiles), 1 one launch */
  int32_t hex_color;        /* TILED: 0 default, 1 colour-sort hex slots even when corner-unique */
  int32_t first_touch;      /* TILED: 0 default (off), 1 first-touch node order inside tiles */
  int32_t allow_nondeterministic; /* must be 1 for tile_mode = shared-memory atomics (5) */
  int32_t lean_kernels;     /* TILED: 0 auto (specialised batch loops for tet-only colour / hex-only
                               two-row corner-phase tiles), 1 off (the general kernel) */
  int32_t resident_sync;    /* resident path: 0 default (stamped halo words, no grid barrier; a runaway
                               call is replayed up to the failing step), 1 grid barrier per step */
} fh_options;

typedef struct {
  int64_t steps_done;
  int64_t fail_step; /* -1 if none */
  int64_t fail_node; /* original numbering; -1 if none */
  double fail_value;
  double time;       /* state time after the call */
  int64_t step_index;
} fh_report;

int fh_create(const fh_mesh *mesh, const fh_boundary *boundary, const fh_options *opts, fh_engine **out);
int fh_destroy(fh_engine *e);

/* state (original node numbering, float64 on the host side) */
int fh_set_temperature(fh_engine *e, const double *T, int64_t n, int64_t step_index, double time);
int fh_get_temperature(fh_engine *e, double *T, int64_t n);
/* last step's net conduction inflow F (solver.py:352 state.inflow).  EXACT:
 * always kept.  TILED: only after fh_keep_inflow(e, 1); entries of Dirichlet
 * nodes (never updated) are 0. */
int fh_get_inflow(fh_engine *e, double *F, int64_t n);
int fh_keep_inflow(fh_engine *e, int32_t on);
int fh_reset_properties(fh_engine *e);                 /* next step refreshes (TI re-freeze) */

/* advance nsteps explicit steps of size dt (solver.py:348-382 each).  If
 * probes were set, T[probe] is recorded after every step whose new index is
 * a multiple of the probe interval.  Returns FH_ERR_INSTABILITY with the
 * report filled when a step produced a non-finite or runaway temperature; the
 * state is then the one right after that step. */
int fh_step(fh_engine *e, int64_t nsteps, double dt, fh_report *rep);

/* fh_step with CUDA events recorded on the engine's stream around the
 * launches; *elapsed_ms = device time of the nsteps steps. */
int fh_step_timed(fh_engine *e, int64_t nsteps, double dt, fh_report *rep, float *elapsed_ms);

/* benchmark variant for working sets that fit in L2: before each of the
 * nsteps steps, `scratch` (device memory, scratch_bytes > L2) is overwritten
 * on the engine's stream; *elapsed_ms = the sum of the per-step device times
 * (the overwrites excluded). */
int fh_step_timed_flush(fh_engine *e, int64_t nsteps, double dt, void *scratch, size_t scratch_bytes,
                        fh_report *rep, float *elapsed_ms);

/* same, with host I/O around it: upload T_in (n doubles), step, download
 * the new field into T_out -- the reference's ExplicitEngine.step contract
 * with host-resident state (used for the e2e measurement). */
int fh_step_host(fh_engine *e, const double *T_in, double *T_out, int64_t n, int64_t nsteps, double dt,
                 fh_report *rep);

/* fh_step_host, double-buffered (single GPU).  Queues: upload T_in into the
 * device staging field of `slot` (0 or 1) on a copy stream, nsteps steps on
 * the engine stream, download of the new field into T_out on a second copy
 * stream; returns without waiting.  T_in / T_out must be pinned and stay
 * untouched until fh_host_wait(slot).  Alternating slots lets the upload of
 * call k+1 and the download of call k share the bus in both directions.  A
 * runaway step is reported by fh_host_wait (FH_ERR_INSTABILITY, fail_step). */
int fh_step_host_async(fh_engine *e, const double *T_in, double *T_out, int64_t n, int64_t nsteps, double dt,
                       int32_t slot);
int fh_host_wait(fh_engine *e, int32_t slot, fh_report *rep);

/* set the static extra nodal power (W, original numbering, n == V) */
int fh_set_q_static(fh_engine *e, const double *q, int64_t n);

/* replace the time-dependent volumetric sources (n <= 8) after creation */
int fh_set_sources(fh_engine *e, const fh_source *sources, int32_t n);

int fh_set_probes(fh_engine *e, const int64_t *nodes, int64_t n, int64_t interval, int64_t capacity);
int fh_get_probes(fh_engine *e, double *values, int64_t max_records, int64_t *n_records);

/* solver.py:384-405 Gershgorin bound 2/lambda_hat at field T (NULL = current
 * state); bitwise == reference in EXACT mode. */
int fh_critical_dt(fh_engine *e, const double *T, int64_t n, double *out);

/* solver.py:223-240 scatter_loads with a given kbar (EXACT mode only). */
int fh_scatter_loads(fh_engine *e, const double *kbar, const double *T, int64_t n, double *out);

/* precompute results (original numbering): lumped node volumes (V) and
 * element volumes (E). */
int fh_get_precompute(fh_engine *e, double *node_volumes, double *elem_volumes);

/* layout facts for the roofline: bytes the step kernel streams per step and
 * counts. */
typedef struct {
  int64_t n_parts, n_slots, n_nodes_owned, n_elements;
  int64_t step_bytes;      /* bytes the fused step streams from/to HBM (layout) */
  int64_t canonical_bytes; /* SURVEY 8(d) canonical bytes per step */
  int32_t kernels_per_step; /* launches per step; 0: the resident EXACT kernel runs many steps per launch */
  int32_t max_part_nodes;
  int32_t resident_ctas;    /* EXACT: CTAs of the resident kernel (0: two launches per step) */
  int32_t resident_threads; /* threads per resident CTA */
} fh_layout;
int fh_get_layout(fh_engine *e, fh_layout *out);

/* raw stream handle (cudaStream_t as void*) for CUDA-event timing from the host */
void *fh_stream(fh_engine *e);

/* permutation new->original node ids (TILED), for bookkeeping tests */
int fh_get_node_order(fh_engine *e, int64_t *new_to_old, int64_t n);

/* multi-GPU: NCCL bootstrap.  Rank 0 creates the id (128 bytes), the
 * caller broadcasts it (torch.distributed), every rank attaches. */
int fh_nccl_unique_id(char *id128);
/* NCCL is loaded with dlopen the first time it is needed: a libnccl.so.2 the
 * process already holds, else `path` (if set here), else the sonames
 * libnccl.so.2 / libnccl.so.  A host that later loads a framework bundling its
 * own NCCL (PyTorch) should name that file here, so that the one NCCL in the
 * process is the version the framework was built against. */
int fh_nccl_library(const char *path);
/* world == 1 builds a one-rank communicator (the fail-flag all-reduce then
 * goes through NCCL): a single-GPU check of the NCCL loading and init path */
int fh_attach_nccl(fh_engine *e, const char *id128, int32_t rank, int32_t world);

/* Host transport for the multi-GPU halo exchange (instead of NCCL, e.g. over
 * gloo or MPI on the host).  fh_step then runs the same per-step schedule --
 * interior tiles, boundary tiles, pack kernel -- copies the packed values to
 * host memory, calls exchange() (blocking), copies the received values back
 * and runs the unpack kernel.  Buffers hold elem_bytes-sized values (4 or 8)
 * grouped by peer, offsets in values (n_peers + 1 entries each).
 * allreduce_min_u64 replaces *value by the minimum over all ranks (fail-flag
 * agreement and the instability report).  Callbacks return 0 on success. */
typedef struct {
  void *ctx;
  int32_t (*exchange)(void *ctx, int32_t n_peers, const int32_t *peers, const void *send, const int64_t *send_offs,
                      void *recv, const int64_t *recv_offs, int32_t elem_bytes);
  int32_t (*allreduce_min_u64)(void *ctx, uint64_t *value);
} fh_transport;
int fh_attach_transport(fh_engine *e, const fh_transport *transport);

/* Halo bookkeeping of a multi-domain engine (rank = domain_lo / width, world =
 * n_domains / width).  Node ids in the original numbering; per-peer ranges
 * [offs[q], offs[q+1]).  fh_halo_export/import move the current halo values
 * through host memory: the exchange used when several ranks share one GPU
 * (tests), where kernels must never wait on one another. */
int fh_halo_info(fh_engine *e, int32_t *world, int32_t *rank, int32_t *n_peers, int64_t *n_send, int64_t *n_recv,
                 int64_t *n_boundary_parts, int64_t *n_parts);
int fh_halo_lists(fh_engine *e, int32_t *peers, int64_t *send_offs, int64_t *send_nodes, int64_t *recv_offs,
                  int64_t *recv_nodes);
int fh_halo_export(fh_engine *e, double *send_values);
int fh_halo_import(fh_engine *e, const double *recv_values);
int fh_get_owned(fh_engine *e, uint8_t *mask, int64_t n);

/* Host-only partition plan (no GPU needed): the tile / domain / halo
 * bookkeeping fh_create performs, for checking it bit for bit.  info[] =
 * {n_parts, parts of rank, boundary parts of rank, peers, n_send, n_recv,
 * node_lo, node_hi, corner_unique, max_phase_tet, max_phase_hex, n_slots,
 * max_local_nodes, colored_ok, max_colors, max_nph_tet, max_nph_hex,
 * sum of tet batch phases, tet batch count (array length), same two for hexes}. */
typedef struct fh_plan fh_plan;
int fh_plan_create(const fh_mesh *mesh, const fh_boundary *boundary, const fh_options *opts, int32_t world,
                   int32_t rank, fh_plan **out);
int fh_plan_info(fh_plan *plan, int64_t *info, int32_t n_info);
int fh_plan_arrays(fh_plan *plan, int64_t *new_to_old, int64_t *part_node_start, int32_t *peers, int64_t *send_offs,
                   int64_t *send_nodes, int64_t *recv_offs, int64_t *recv_nodes);
int fh_plan_destroy(fh_plan *plan);

/* ------------------------------------------------------------------ */
/* 3. Mesh ingest and text output (host only, no GPU)                   */
/* ------------------------------------------------------------------ */

/* mesh.py:192-236 parse_mesh_text: the reference's mesh grammar (nodes /
 * elements tet4|hex8 / nodeset blocks, '#' comments, Python splitlines() line
 * breaks and split() whitespace over UTF-8 text).  Tokens convert like
 * Python int()/float() (underscores, inf/nan; floats correctly rounded).
 * On a grammar error returns FH_ERR_FORMAT with the reference's message
 * (without the "line N: " prefix) and *err_line = the 1-based line the
 * reference reports.  Geometry is not validated here (Mesh() does it).
 * n_threads <= 0: all hardware threads convert the coordinate block. */
typedef struct fh_mesh_text fh_mesh_text;
int fh_mesh_parse(const char *text, int64_t len, int32_t n_threads, fh_mesh_text **out, int64_t *err_line);
int fh_mesh_text_info(fh_mesh_text *m, int64_t *n_nodes, int64_t *n_tets, int64_t *n_hexes, int32_t *n_sets);
/* nodes (V,3) f64, tets (Et,4), hexes (Eh,8) i64 in file order; NULL skips */
int fh_mesh_text_arrays(fh_mesh_text *m, double *nodes, int64_t *tets, int64_t *hexes);
/* node set i (file order): name (NUL-terminated), members in file order;
 * ids == NULL only reports *count */
int fh_mesh_text_set(fh_mesh_text *m, int32_t i, char *name, int64_t name_cap, int64_t *ids, int64_t *count);
int fh_mesh_text_destroy(fh_mesh_text *m);

/* Text rows as the reference writes them (mesh.py:241-253 serialize_mesh_text,
 * vtkio.py:20-52 vtk_text, cli.py:81-86 probes.csv): each row is row_prefix
 * (may be NULL), then `cols` values joined by `sep`, then '\n'.  Doubles are
 * Python repr(float) (shortest round-trip digits), integers str(int).  With
 * out == NULL only *used (the byte count) is computed. */
int fh_format_f64(const double *v, int64_t rows, int64_t cols, char sep, const char *row_prefix, int32_t n_threads,
                  char *out, int64_t cap, int64_t *used);
int fh_format_i64(const int64_t *v, int64_t rows, int64_t cols, char sep, const char *row_prefix, int32_t n_threads,
                  char *out, int64_t cap, int64_t *used);

#ifdef __cplusplus
}
#endif
#endif
