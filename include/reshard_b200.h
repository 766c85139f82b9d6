/*
 * reshard_b200.h — C ABI of the B200-native resharding path (libreshard_b200.so).
 *
 * Drop-in boundary for the reference's planner + transition engine. The reference
 * exposes a header-only C++ API in namespace reshard (/root/reference/proj/include/
 * reshard); every entry point below names the reference interface it replaces.
 * The same C++ API is also shipped, re-implemented, under
 * paper_2605_18815_b200/csrc/reshard/ for C++ callers.
 *
 * Conventions: plain pointers and sizes only; every function returns an int status
 * (RS_OK = 0) and never throws; rs_last_error() gives the thread-local message of
 * the last failure. Objects are created and destroyed by the library; the caller
 * owns device buffers it binds with rs_exec_bind(). Planner calls are reentrant
 * (SPEC.md:252-253); an rs_exec_t is driven by one host thread.
 */
#ifndef RESHARD_B200_H
#define RESHARD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (SPEC.md:523 exit codes 0/1/2 map to OK / VIOLATION / CONFIG) */
#define RS_OK 0
#define RS_ERR_VIOLATION 1 /* verification found mismatching elements */
#define RS_ERR_CONFIG 2    /* reference ConfigError (common.hpp:30-33): bad input */
#define RS_ERR_INTERNAL 3  /* reference std::logic_error: broken invariant */
#define RS_ERR_CUDA 4      /* CUDA runtime / driver failure (incl. no GPU) */
#define RS_ERR_NCCL 5
#define RS_ERR_BUDGET 6    /* memory-aware schedule infeasible under the HBM cap */

/* ---- state kinds (common.hpp:37 StateKind order) and buffers */
#define RS_KIND_PARAM 0
#define RS_KIND_OPTIM 1
#define RS_KIND_GRAD 2
#define RS_KIND_SCALAR 3

#define RS_BUF_PARAM 0   /* params, dtype_bytes per element, local_layout order */
#define RS_BUF_MASTER 1  /* fp32 master weights (optimizer shard) */
#define RS_BUF_M 2       /* fp32 Adam m */
#define RS_BUF_V 3       /* fp32 Adam v */
#define RS_BUF_GRAD 4    /* fp32 grads, param geometry (GradientPolicy::Migrate only) */
#define RS_BUF_SCALARS 5 /* scalar_words x u64 */

#define RS_SIDE_SRC 0
#define RS_SIDE_DST 1

typedef struct rs_model rs_model_t;
typedef struct rs_plan rs_plan_t;
typedef struct rs_exec rs_exec_t;

/* TensorSpec (model.hpp:30-44). tp_axis / expert_axis: -1 = none. */
typedef struct {
    const char* id;
    int ndim; /* 1..4 */
    int64_t shape[4];
    int layer;
    int tp_axis;
    int expert_axis;
    int dtype_bytes;
} rs_tensor_t;

/* ParallelConfig (parallel.hpp:28-46). order NULL -> "pp-dp-tp". */
typedef struct {
    int dp, tp, pp, ep;
    int zero;
    const char* order;
} rs_cfg_t;

/* WorldMap (worldmap.hpp:30-39). */
typedef struct {
    int n_src;
    const int* src_phys;
    int n_dst;
    const int* dst_phys;
} rs_worldmap_t;

/* Topology (topology.hpp:25-31); only the node grouping feeds the planner. */
typedef struct {
    int num_nodes;
    int ranks_per_node;
} rs_topo_t;

/* PlanOptions (routing.hpp:40-44) + the D2 extension switch. */
typedef struct {
    int migrate_grads;     /* GradientPolicy::Migrate */
    int balance_fanout;
    int64_t scalar_words;
    int allow_oversourced; /* extension: resolve over-sourced ZeRO intervals (reference throws) */
} rs_options_t;

/* SliceTransfer (routing.hpp:50-77) as POD. flat=1: [lo[0],hi[0]) global flat run. */
typedef struct {
    int kind, tensor, flat, ndim;
    int64_t lo[4], hi[4];
    int src_rank, dst_rank, src_phys, dst_phys;
    int64_t count, bytes;
} rs_transfer_t;

typedef struct {
    int64_t num_transfers;   /* RoutingPlan::transfers.size() */
    int64_t bytes_moved;     /* RoutingPlan::bytes_moved() routing.hpp:151-156 */
    int64_t bytes_retained;  /* RoutingPlan::bytes_retained() routing.hpp:157-169 */
    int64_t num_box_transfers, num_flat_transfers, num_triples;
    int src_world, dst_world, num_participants;
    int64_t total_numel;
    uint64_t fingerprint;    /* ModelSpace::fingerprint() */
} rs_plan_summary_t;

const char* rs_last_error(void);
const char* rs_version(void);
/* one process driving several GPUs: let `device` store into `peer`'s memory directly
 * (cudaDeviceEnablePeerAccess; already-enabled is not an error) */
int rs_enable_peer_access(int device, int peer);
void rs_free(void* p);

/* build_model_space (model.hpp:127-144), validate_model (model.hpp:95-123) */
int rs_model_create(const rs_tensor_t* tensors, int n, int num_layers, int num_experts, rs_model_t** out);
void rs_model_destroy(rs_model_t* m);

/* plan_parameters + plan_optimizer + plan_scalars + resolve_peers
 * (routing.hpp:231, :287, :341, :360), with validate_config x2 first.
 * wm / topo / opts may be NULL (identity map, 1 node x 8, defaults). The plan keeps a
 * reference to the model: destroy the plan first. */
int rs_plan_create(const rs_model_t* m, const rs_cfg_t* src, const rs_cfg_t* dst, const rs_worldmap_t* wm,
                   const rs_topo_t* topo, const rs_options_t* opts, rs_plan_t** out);
/* same, from scenario text; the plan owns its model */
int rs_plan_from_scenario(const char* text, int allow_oversourced, rs_plan_t** out);
void rs_plan_destroy(rs_plan_t* p);
int rs_plan_summary(const rs_plan_t* p, rs_plan_summary_t* out);
/* format_transfer lines (routing.hpp:86-90) in transfer_order_less order
 * (routing.hpp:79-84). device < 0: host expansion; >= 0: GPU planner on that device. */
int rs_plan_dump(const rs_plan_t* p, int device, char** out, size_t* len);
/* resolved transfer list (reference SliceTransfers), same order as rs_plan_dump */
int rs_plan_transfers(const rs_plan_t* p, int device, rs_transfer_t** out, int64_t* n);
/* project / local_layout / project_optimizer of every rank of one side
 * (project.hpp:44, :94, :146), text lines */
int rs_plan_regions(const rs_plan_t* p, int side, char** out, size_t* len);
/* per-GPU byte accounting under contiguous-block placement of the plan's devices on
 * n_gpus GPUs (host only): local copies, bytes pushed to / received from peers */
typedef struct {
    int64_t local_bytes, out_bytes, in_bytes, ops;
} rs_placement_stats_t;
/* ---- state layout of one virtual rank (the buffer contract): what a
 * training job needs to register its tensors as views into the transition buffers
 * (PAPER.md:938-939). side: RS_SIDE_SRC / RS_SIDE_DST. */
typedef struct {
    int tensor;                  /* index in the model's declaration order */
    int expert;                  /* 1: lives in the expert span */
    int64_t box_lo[4], box_hi[4];/* the rank's box of the tensor (tensor coordinates) */
    int64_t local_lo, local_hi;  /* element range in its span (dense or expert) */
    int64_t param_byte_off;      /* byte offset in the param buffer */
    int64_t elem_off;            /* element offset in the param-geometry buffers (grads) */
} rs_segment_t;
typedef struct {
    int phys, n_segments;
    int64_t dense_len, expert_len;          /* elements */
    int64_t dshard_lo, dshard_hi;           /* ZeRO shard of the dense span (whole span without ZeRO) */
    int64_t eshard_lo, eshard_hi;           /* ... of the expert span */
    int64_t param_bytes, nelem, optim_len;  /* optimizer buffers: [dense shard | expert shard], fp32 each */
    int64_t scalar_bytes;                   /* scalar blob (scalar_words x 8 B) */
} rs_rank_geom_t;
int rs_plan_rank_geom(const rs_plan_t* p, int side, int rank, rs_rank_geom_t* out);
int rs_plan_segments(const rs_plan_t* p, int side, int rank, rs_segment_t* out, int cap, int* n);
/* tensor `index` of the model: id (NUL-terminated into id_buf), shape, dtype bytes */
int rs_plan_tensor(const rs_plan_t* p, int index, char* id_buf, int cap, int64_t shape[4], int* ndim, int* dtype_bytes);
int rs_plan_num_tensors(const rs_plan_t* p, int* n);

int rs_plan_placement(const rs_plan_t* p, int n_gpus, int gpu, rs_placement_stats_t* out);
/* copy bytes between physical devices: out[s * n + d] (n = *n_phys, highest participating
 * phys + 1; fills when cap >= n * n). Off-diagonal entries sum to bytes_moved; the
 * diagonal holds on-device copies. Input of the co-location search when devices share a GPU
 * (no reference counterpart: the reference runs one device per GPU). */
int rs_plan_traffic(const rs_plan_t* p, int64_t* out, int cap, int* n_phys);
/* participating physical devices, ascending (WorldMap::participants, worldmap.hpp:60-68);
 * *n = count (fills at most cap) */
int rs_plan_participants(const rs_plan_t* p, int* phys, int cap, int* n);
/* validate_plan: invariants + destination coverage; violations are
 * returned (one per line), not raised. drop >= 0 removes one fragment first (fault
 * injection: box transfers are indexed first, then ZeRO runs). */
int rs_plan_validate(const rs_plan_t* p, int64_t drop, char** report, size_t* len, int64_t* n_violations);
/* host expansion of the ZeRO runs with the GPU planner's per-row algorithm (tests) */
/* the GPU box planner (batched (dst rank, tensor, src rank) intersections) on `device`:
 * kernel milliseconds, number of box transfers, and whether they equal the host plan's */
int rs_plan_box_routes_timed(const rs_plan_t* p, int device, double* ms, int64_t* n_boxes, int* equal_host);
int rs_plan_dump_rows_host(const rs_plan_t* p, char** out, size_t* len);
/* expand the ZeRO optimizer transfers (1.84 M runs for Llama-3-8B) and report the
 * time: device >= 0 -> GPU planner kernels (ms of device time), < 0 -> host sweep */
int rs_plan_expand_timed(const rs_plan_t* p, int device, double* ms, int64_t* n_runs);

/* ---- Elastic Device Manager support */
#define RS_GROUP_DP 0
#define RS_GROUP_TP 1
#define RS_GROUP_PP 2
#define RS_GROUP_EP 3
#define RS_GROUP_EDP 4
/* get_or_create_groups' pure derivation: communicator groups of cfg
 * along one dimension; out[g * group_size + k] = k-th rank of group g. */
int rs_config_groups(const rs_cfg_t* cfg, int dim, int* out, int cap, int* n_groups, int* group_size);
/* rank_coord (parallel.hpp:88-106): {pp, dp, tp, ep, edp} */
int rs_rank_coord(const rs_cfg_t* cfg, int rank, int coord[5]);

/* ---- transition schedule: Algorithm 1 */
typedef struct rs_schedule rs_schedule_t;
typedef struct {
    int num_devices;       /* N = participants */
    int num_stages;
    int num_collectives;
    int num_steps;         /* steps with traffic */
    int64_t budget;        /* M_global_min = min(mem_avail) */
    int64_t p2p_bytes, collective_bytes;
    int64_t num_fragments;
} rs_schedule_summary_t;
#define RS_COMM_P2P 0
#define RS_COMM_BROADCAST 1
#define RS_COMM_SCATTER 2
#define RS_COMM_GATHER 3
/* xor_schedule: peer of device i at step s, or -1 */
/* ---- Elastic Device Manager: cached communicator
 * groups per configuration, the side thread preparing the next world, the accounting. */
typedef struct rs_edm rs_edm_t;
typedef struct {
    double init_s, overlapped_s, switch_s, exposed_s, ratio; /* ratio -1: undefined */
} rs_edm_accounting_t;
#define RS_EDM_BLOCKING 0
#define RS_EDM_OVERLAPPED 1
#define RS_EDM_IN_PLACE 2
int rs_edm_create(rs_edm_t** out);
void rs_edm_destroy(rs_edm_t* e);
/* get_or_create_groups for one dimension (cached; *cache_hit = 1 when it was) */
int rs_edm_groups(rs_edm_t* e, const rs_cfg_t* cfg, int dim, int* out, int cap, int* n_groups, int* group_size,
                  int* cache_hit);
int rs_edm_cache_stats(const rs_edm_t* e, int64_t* hits, int64_t* misses, double* creation_s);
/* run build(arg) on a side thread (new world's plan, executor, buffers, peer mappings) */
int rs_edm_prepare_async(rs_edm_t* e, int (*build)(void* arg), void* arg);
int rs_edm_ready(const rs_edm_t* e, int* ready);
/* join the side thread: its preparation time and build's return code */
int rs_edm_wait(rs_edm_t* e, double* init_s, int* build_rc);
/* simulate_scale_event accounting: window_s >= 0 = measured overlap window, else whole
 * training steps of train_step_s fit into init_s */
int rs_edm_accounting(double init_s, double switch_s, double window_s, double train_step_s, int mode,
                      rs_edm_accounting_t* out);
/* New-world NCCL communicators built natively: a fresh unique id (rank 0
 * of the new world draws it, the caller broadcasts the 128 bytes), then the world
 * communicator (ncclCommInitRankConfig, blocking = 0) and one ncclCommSplit per dimension
 * (colors[RS_DIM_*] < 0: skip), polled to completion on the calling thread — the EDM side
 * thread. Cached per configuration (*cache_hit). libnccl.so.2 is loaded at run time. */
#define RS_NCCL_ID_BYTES 128
int rs_nccl_unique_id(void* out, size_t cap);
int rs_nccl_version(char* out, size_t cap);
int rs_edm_comm_create(rs_edm_t* e, const rs_cfg_t* cfg, const void* uid, int nranks, int rank, int device,
                       const int colors[5], int* cache_hit, double* init_s, double* split_s);
/* the ncclComm_t of dimension `dim` (-1: world) of a created configuration, or NULL */
int rs_edm_comm_get(rs_edm_t* e, const rs_cfg_t* cfg, int dim, void** comm);
/* all-reduce (sum) of one 1.0f over that communicator on `stream`: *sum = its size */
int rs_edm_comm_check(rs_edm_t* e, const rs_cfg_t* cfg, int dim, void* stream, float* sum);
int rs_edm_comm_destroy(rs_edm_t* e, const rs_cfg_t* cfg);

int rs_xor_peer(int i, int s, int n);
/* MemoryAwareChunk: stage index per step (steps ascending, cost[k]
 * for steps[k]); RS_ERR_BUDGET if one step exceeds min(mem_avail) */
int rs_memory_aware_chunk(const int* steps, const int64_t* cost, int n_steps, const int64_t* mem_avail, int n_ranks,
                          int* stage_of_step, int64_t* budget);
/* build_schedule. mem_avail: per device (NULL = unbounded). */
int rs_schedule_build(const rs_plan_t* p, const int64_t* mem_avail, int n, int promote, rs_schedule_t** out);
void rs_schedule_destroy(rs_schedule_t* s);
int rs_schedule_summary(const rs_schedule_t* s, rs_schedule_summary_t* out);
/* stage k: its steps and mem_cost */
int rs_schedule_stage(const rs_schedule_t* s, int k, int* steps, int cap, int* n, int64_t* mem_cost);
/* device dev in stage k, step index q: peer (-1 inactive) and buffer sizes */
int rs_schedule_peer(const rs_schedule_t* s, int k, int q, int dev, int* peer, int64_t* send_bytes, int64_t* recv_bytes);
/* collective c: kind, root, bytes, participants */
int rs_schedule_collective(const rs_schedule_t* s, int c, int* kind, int* root, int64_t* bytes, int* participants, int cap,
                           int* n);
int rs_schedule_dump(const rs_schedule_t* s, char** out, size_t* len);

/* ---- executor: Algorithm 1 ExecuteSwitch / SPEC execute
 * (SPEC.md:375-383), push model over NVLink. One rs_exec_t per GPU/process. */
typedef struct {
    int n_gpus;            /* GPUs the plan's physical devices are placed on (contiguous blocks) */
    int gpu;               /* this process's GPU index */
    int device;            /* CUDA device ordinal */
    int with_grads;        /* allocate/migrate grad buffers */
    int64_t tile_bytes;    /* 0 -> default */
    int ctas_per_sm;       /* 0 -> default */
} rs_exec_opts_t;

typedef struct {
    int64_t local_bytes;   /* bytes copied within this GPU's HBM (incl. retained) */
    int64_t remote_bytes;  /* bytes stored into peer GPUs over NVLink */
    int64_t tiles;
    int64_t tiles_by_class[5];
    int64_t launches;      /* kernel launches per rs_exec_run */
    int64_t mc_bytes;      /* bytes delivered to peers by NVLS multicast stores */
    int64_t dup_bytes;     /* replica bytes copied on this GPU by rs_exec_run_dup */
    int64_t scatter_bytes; /* bytes of promoted Scatter collectives this GPU pushes as their root */
    int64_t gather_bytes;  /* bytes of promoted Gather collectives this GPU pulls as their root */
} rs_exec_stats_t;

/* ---- memory-aware arena (Algorithm 1 FreeObsoleteBuffers / eager free,
 * PAPER.md:668,689,942): old (A) and new (B) layouts of every virtual rank on one GPU
 * in CUDA VMM ranges; B chunks reuse the physical memory of A chunks that die in an
 * earlier stage (for a round trip, also vice versa). plan_ba may be NULL (one way). */
typedef struct rs_arena rs_arena_t;
typedef struct {
    int64_t physical_bytes, a_bytes, b_bytes, aliased_bytes, chunks;
    int64_t stage_groups[2]; /* concurrent stage groups (barriers) per direction */
    int64_t bands;           /* layer bands per destination rank in the stage units */
} rs_arena_stats_t;
int rs_arena_create(const rs_plan_t* plan_ab, const rs_plan_t* plan_ba, int device, int64_t cap_bytes,
                    int64_t chunk_bytes, int with_grads, rs_arena_t** out);
void rs_arena_destroy(rs_arena_t* a);
/* layout 0 = A (src of plan_ab), 1 = B (dst of plan_ab) */
int rs_arena_buffer(const rs_arena_t* a, int layout, int rank, int buf, void** dptr, int64_t* bytes);
/* stage order of direction 0 (A->B) or 1 (B->A): units rank * bands + layer band */
int rs_arena_stage_order(const rs_arena_t* a, int dir, int* out, int cap, int* n);
/* per position of that order: 1 = a barrier must precede it (positions between two cuts
 * share one stage and run concurrently); position 0 is always 1 */
int rs_arena_stage_cuts(const rs_arena_t* a, int dir, int* out, int cap, int* n);
int rs_arena_stats(const rs_arena_t* a, rs_arena_stats_t* out);
/* FreeObsoleteBuffers at run time (one-way arenas on one GPU): once
 * stage `stage` of the transition has completed, unmap every old-layout chunk last read in
 * a stage <= `stage` and return the physical chunks the new layout does not reuse to the
 * driver (cuMemUnmap + cuMemRelease). *freed: bytes released by this call. */
int rs_arena_release_through(rs_arena_t* a, int stage, int64_t* freed);
/* host-only memory plan (no GPU): stats and the execution-simulation check
 * (violations == 0 means every read sees its own data) */
/* fewest concurrency groups of the stage order whose memory plan for `gpu` fits
 * cap_bytes (*groups = -1: none); every GPU must use the same groups (take the max) */
int rs_memory_min_groups(const rs_plan_t* plan_ab, const rs_plan_t* plan_ba, int64_t chunk_bytes, int with_grads,
                         int n_gpus, int gpu, int64_t cap_bytes, int* groups, int64_t* physical_bytes);
/* the same for the buffers GPU `gpu` of n_gpus hosts, with the stage order coarsened
 * into `groups` concurrency groups (0 = one per stage) */
int rs_memory_plan_ex(const rs_plan_t* plan_ab, const rs_plan_t* plan_ba, int64_t chunk_bytes, int with_grads, int n_gpus,
                      int gpu, int groups, int bands, rs_arena_stats_t* stats, int64_t* violations, int* order_ab,
                      int* order_ba, int cap);
/* the schedule ladder (arena.hpp schedule_levels): the first level whose plan for `gpu`
 * fits cap_bytes (*level = -1: none); rs_memory_schedule_level gives its (bands, groups),
 * groups -1 = rounds (one unit per GPU per group) */
int rs_memory_schedule(const rs_plan_t* plan_ab, const rs_plan_t* plan_ba, int64_t chunk_bytes, int with_grads, int n_gpus,
                       int gpu, int64_t cap_bytes, int* level, int64_t* physical_bytes);
int rs_memory_schedule_level(const rs_plan_t* plan_ab, int n_gpus, int level, int* bands, int* groups);
/* physical bytes GPU `gpu` needs at every level of the ladder (*n = number of levels):
 * across GPUs, take the first level whose footprint fits on every rank */
int rs_memory_schedule_footprints(const rs_plan_t* plan_ab, const rs_plan_t* plan_ba, int64_t chunk_bytes, int with_grads,
                                  int n_gpus, int gpu, int64_t* out, int cap, int* n);
/* the same ladder with each level's modeled seconds (per stage group: the busiest GPU's
 * NVLink / HBM bound plus a barrier; both directions): pick the fastest level that fits
 * the cap on every GPU */
int rs_memory_schedule_costs(const rs_plan_t* plan_ab, const rs_plan_t* plan_ba, int64_t chunk_bytes, int with_grads,
                             int n_gpus, int gpu, int64_t* bytes, double* seconds, int cap, int* n);
/* the plan's stage cuts of direction `dir` (1 = a barrier precedes that position) */
int rs_memory_plan_cuts(const rs_plan_t* plan_ab, const rs_plan_t* plan_ba, int64_t chunk_bytes, int with_grads,
                        int n_gpus, int gpu, int groups, int bands, int dir, int* cuts, int cap, int* n);
int rs_memory_plan(const rs_plan_t* plan_ab, const rs_plan_t* plan_ba, int64_t chunk_bytes, int with_grads,
                   rs_arena_stats_t* stats, int64_t* violations, int* order_ab, int* order_ba, int cap);
/* multi-GPU arena: this process maps the buffers of the virtual ranks placed on GPU
 * `gpu` of `n_gpus` (shareable VMM); peers' buffers are imported from their export */
int rs_arena_create_multi(const rs_plan_t* plan_ab, const rs_plan_t* plan_ba, int n_gpus, int gpu, int device,
                          int64_t cap_bytes, int64_t chunk_bytes, int with_grads, int groups, int bands,
                          rs_arena_t** out);
/* POSIX-FD export of this GPU's physical allocations + mapping table (malloc'd; rs_free) */
int rs_arena_export(const rs_arena_t* a, int** fds, int* n_fds, void** table, size_t* table_len);
/* map a peer's buffers (consumes the descriptors) */
int rs_arena_import(rs_arena_t* a, const int* fds, int n_fds, const void* table, size_t table_len);
/* descriptor exchange between local processes (Unix socket, SCM_RIGHTS, abstract name) */
int rs_fdx_listen(const char* name, int* sock);
int rs_fdx_send(const char* peer_name, const int* fds, int n_fds, const void* payload, size_t len);
int rs_fdx_recv(int sock, int** fds, int* n_fds, void** payload, size_t* len);
int rs_fdx_close(int fd);
/* memory-aware stages across GPUs: one stage per call, barrier in between (caller) */
int rs_exec_num_stages(const rs_exec_t* e, int* n);
int rs_exec_run_stage(rs_exec_t* e, int stage, void* stream, int* launches);
/* run the plan as memory-aware stages: dst ranks in the given order */
int rs_exec_set_stages(rs_exec_t* e, const int* dst_order, int n);
/* rs_exec_run replayed from a CUDA graph (captured at the first call after each prepare,
 * per stream): small transitions are launch-bound */
int rs_exec_run_graph(rs_exec_t* e, void* stream, int* launches);
/* the same order, grouped: cuts[i] == 1 starts a new stage at position i (cuts may be NULL) */
int rs_exec_set_stage_groups(rs_exec_t* e, const int* dst_order, const int* cuts, int n);

/* ---- broadcast promotion over NVLS multicast (optimize_primitives, SPEC.md:282-290,
 * PAPER.md:719-740). A group = one source region copied to >= 2 destination ranks on
 * distinct GPUs at the source's own offsets (DP replicas); slot s = each GPU's s-th
 * destination rank. The root GPU stores it once through a multicast address whose object
 * binds the root's source buffer and every member's destination buffer. */
#define RS_MAX_MEMBERS 64
typedef struct {
    int id, root_rank, root_gpu, buf, slot, n_members;
    int member_gpu[RS_MAX_MEMBERS], member_rank[RS_MAX_MEMBERS];
    int64_t buffer_bytes;  /* size of buffer `buf` (equal on root and members) */
    int64_t payload_bytes; /* bytes the root stores once */
} rs_bcast_group_t;
int rs_exec_bcast_groups(rs_exec_t* e, rs_bcast_group_t* out, int cap, int* n);
/* root only; mc_va NULL reverts to per-destination pushes; takes effect at the next prepare */
int rs_exec_set_multicast(rs_exec_t* e, int id, void* mc_va);
/* replica dedup: a region bound for several replica ranks on one GPU crosses NVLink once;
 * after rs_exec_run on every GPU and a barrier, rs_exec_run_dup copies the other replicas.
 * on = 2 (early): stage 1 is a tail of the other pushes sized to hide the copies, stage 0
 * the rest incl. the primaries (rs_exec_num_stages = 2): run stage 0, barrier on it, then rs_exec_run_dup on a second
 * stream overlaps stage 1. Needs a single memory stage. */
int rs_exec_set_replica_dedup(rs_exec_t* e, int on);
int rs_exec_run_dup(rs_exec_t* e, void* stream, int* launches);

typedef struct rs_mc rs_mc_t;
int rs_mc_create(int64_t bytes, int n_devices, rs_mc_t** out);
int rs_mc_import(int fd, int64_t bytes, rs_mc_t** out); /* consumes fd */
int rs_mc_export(const rs_mc_t* m, int* fd);
int rs_mc_add_device(rs_mc_t* m, int device);
/* every member must have added its device first (the bind blocks until then) */
int rs_mc_bind_arena(rs_mc_t* m, const rs_arena_t* a, int layout, int rank, int buf);
int rs_mc_map(rs_mc_t* m, int device, void** mc_va);
void rs_mc_destroy(rs_mc_t* m);
int rs_arena_bind_size(const rs_arena_t* a, int layout, int rank, int buf, int64_t* bytes);

/* one shareable VMM device buffer (POSIX-FD handle): state buffers that peers map
 * without cudaIpc and a multicast object can bind. Import maps a peer's buffer for
 * `device` (consumes fd). The size is rounded up to the VMM granularity (2 MiB). */
typedef struct rs_vmm rs_vmm_t;
int rs_vmm_alloc(int device, int64_t bytes, rs_vmm_t** out);
int rs_vmm_import(int fd, int64_t bytes, int device, rs_vmm_t** out);
int rs_vmm_export(const rs_vmm_t* v, int* fd);
int rs_vmm_ptr(const rs_vmm_t* v, void** ptr, int64_t* mapped_bytes);
void rs_vmm_free(rs_vmm_t* v);
int rs_mc_bind_vmm(rs_mc_t* m, const rs_vmm_t* v, int64_t mc_offset);

int rs_exec_create(const rs_plan_t* p, const rs_exec_opts_t* o, rs_exec_t** out);

/* SPEC execute in one call, for FFI callers that own their buffers:
 * builds the executor for opts' GPU, binds every listed buffer (this GPU's and the peers'
 * it has mapped), prepares, runs on `stream` and waits. mode: RS_EXEC_FUSED (the push; the
 * staged NCCL comparison and replica dedup need cross-rank steps: use rs_exec_*). */
typedef struct {
    int side, rank, buf;   /* RS_SIDE_*, virtual rank, RS_BUF_* */
    void* ptr;
    int64_t bytes;
} rs_state_buffer_t;
#define RS_EXEC_FUSED 0
int rs_execute(const rs_plan_t* p, const rs_exec_opts_t* o, const rs_state_buffer_t* bufs, int n_bufs, void* stream,
               int mode, int* launches);
void rs_exec_destroy(rs_exec_t* e);
int rs_exec_alloc(rs_exec_t* e);
int rs_exec_bind(rs_exec_t* e, int side, int rank, int buf, void* dptr, int64_t bytes);
int rs_exec_buffer(rs_exec_t* e, int side, int rank, int buf, void** dptr, int64_t* bytes, int* gpu);
int rs_exec_ipc_export(rs_exec_t* e, void* out, size_t cap, size_t* len);
int rs_exec_ipc_import(rs_exec_t* e, const void* blob, size_t len);
int rs_exec_prepare(rs_exec_t* e);
/* Algorithm 1 buffered mode (PackData / AsyncSend+Recv / UnpackData):
 * moves between GPUs go through per-channel contiguous buffers (channel = src phys ->
 * dst phys; layout derived from the plan, identical on both sides); the transport
 * (NCCL send/recv, the measured comparison) is the caller's. Same-GPU moves stay fused. */
int rs_exec_prepare_staged(rs_exec_t* e);
int rs_exec_channel_bytes(const rs_exec_t* e, int src_phys, int dst_phys, int64_t* bytes);
/* per-op packed sizes of a channel (SPEC execute "naive" mode: one message per fragment) */
int rs_exec_channel_ops(const rs_exec_t* e, int src_phys, int dst_phys, int64_t* sizes, int64_t cap, int64_t* n);
int rs_exec_pack(rs_exec_t* e, int src_phys, int dst_phys, void* dbuf, void* stream);
int rs_exec_unpack(rs_exec_t* e, int src_phys, int dst_phys, const void* dbuf, void* stream);
/* load_state on this GPU's ranks of one side */
int rs_exec_fill(rs_exec_t* e, int side, uint64_t seed, void* stream);
int rs_exec_run(rs_exec_t* e, void* stream, int* launches);
/* verify_state on this GPU's ranks of one side */
int rs_exec_verify(rs_exec_t* e, int side, uint64_t seed, void* stream, int64_t* mismatches, int64_t* first_bad);
/* copy `bytes` at `offset` of a buffer this GPU can address into host memory (a result
 * readback; synchronous on `stream`) */
int rs_exec_read(rs_exec_t* e, int side, int rank, int buf, int64_t offset, void* host, int64_t bytes, void* stream);
int rs_exec_stats(const rs_exec_t* e, rs_exec_stats_t* out);
/* ---- SynchronizeAll on the device: a cross-GPU flag barrier enqueued on a
 * stream, so memory-aware stages and consecutive transitions need no host round trip.
 * Each rank creates one, exports its handle, imports every peer's (cudaIpc), then every
 * rank enqueues the same sequence of rs_sync_barrier calls. A spin that exceeds the
 * timeout (20 s) gives up and sets the status rs_sync_status reports. */
typedef struct rs_sync rs_sync_t;
int rs_sync_create(int rank, int world, int device, rs_sync_t** out);
void rs_sync_destroy(rs_sync_t* s);
int rs_sync_export(const rs_sync_t* s, void* out, size_t cap, size_t* len);
int rs_sync_import(rs_sync_t* s, int peer, const void* blob, size_t len);
int rs_sync_barrier(rs_sync_t* s, void* stream);
int rs_sync_status(rs_sync_t* s, int* timed_out);

/* drive the executor's bound buffers with a re-computed plan of the same transition (same
 * configs, world map, model and buffer geometry: RS_ERR_CONFIG otherwise); the next
 * rs_exec_prepare builds descriptors from it. The plan must outlive its use. */
int rs_exec_set_plan(rs_exec_t* e, const rs_plan_t* p);
/* Execute the promoted collectives of optimize_primitives
 * as their own primitives: a Scatter is pushed by its root, a Gather is PULLED by its root
 * (the destination GPU reads every source's slice over NVLink into its contiguous region;
 * one receiver's ingress is the bound and peer loads outrun peer stores there). The
 * source buffers must then be mapped on the destination too: call before
 * rs_exec_ipc_export, on every rank. Takes effect at the next prepare. */
int rs_exec_set_collectives(rs_exec_t* e, int on);
/* GPU index (in [0, n_gpus)) the executor places physical device `phys` on */
int rs_exec_gpu_of_phys(const rs_exec_t* e, int phys, int* gpu);

#ifdef __cplusplus
}
#endif
#endif
