/*
 * mlfabric.h — C ABI of the B200-native MLfabric plan-execution hot path.
 *
 * MLfabric (Viswanathan & Akella, arXiv 1907.00434; /root/reference/PAPER.md,
 * cited P:line) intercepts every worker push, decides per batch an ordering of
 * the updates under the delay bound tau_max, an in-network aggregation
 * partition and a bounded-divergence replica set, then the updates flow to the
 * parameter server in that order (§3; §5).  This library
 * is that data path on one B200 box:
 *
 *   mlf_plan        host C++, pure: Alg. 1-2 ordering, Alg. 3
 *                   aggregation, App. B.2 multi-server
 *                   components, §5.3 replication.
 *   mlf_execute     sm_100a CUDA: for every commit of the plan, in order,
 *                   w <- w - lr * (left fold of the commit's updates), one HBM
 *                   pass over w, each operand read once, the replica mirror
 *                   stored in the same pass (Eq. 2 P:278 with gamma = 0).
 *   mlf_init / mlf_submit_update / mlf_batch_view / mlf_sync /
 *   mlf_pull_model  the PS API around it (Table 1: push with
 *                   update_norm, get; registerAsServer/Replica params tau_max,
 *                   Div_max).
 *
 * Conventions
 *   - Every function returns mlf_status and never throws or aborts; on error
 *     mlf_last_error() (thread-local) describes it, outputs are unspecified and
 *     no device work has been enqueued.
 *   - Times are integer nanoseconds relative to the batch start, sizes are
 *     bytes, rates are bytes/second (reading R8).  Plans are
 *     deterministic and bit-exact across implementations.
 *   - All device memory is allocated by the caller (PyTorch) and borrowed for
 *     the lifetime of the context.  Host arrays passed in are borrowed only for
 *     the duration of the call.
 *   - Planner node ids: the caller numbers the network's nodes; a context maps
 *     worker w to node worker_node[w] (default w) in mlf_batch_view.  On one
 *     B200 box the nodes are the GPUs: the virtual workers multiplexed on a GPU
 *     share its NVLink egress, exactly as the paper's co-located workers share a
 *     host NIC.
 *
 * Readings of silent or ambiguous passages (R1-R25) are listed in DESIGN.md §3.
 */
#ifndef MLFABRIC_H
#define MLFABRIC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MLF_OK = 0,
  MLF_E_INVALID = 1,        /* null pointer, id out of range, duplicate submit, plan inconsistent with the batch */
  MLF_E_STATE = 2,          /* call not legal in the context's current state (slot in flight, ...) */
  MLF_E_CUDA = 3,           /* any CUDA runtime error; sticky, destroy the context */
  MLF_E_UNSCHEDULABLE = 4,  /* an update's path to a server/replica is down forever (R9) */
  MLF_E_CAPACITY = 5        /* caller-provided output arrays too small */
} mlf_status;

typedef enum { MLF_F32 = 0, MLF_BF16 = 1 } mlf_dtype;

/* ======================================================================
 * Planning (pure host C++, reentrant, no CUDA)
 * ====================================================================== */

/* The network G = (V, E) of App. B.1 in the per-node NIC model the
 * evaluation uses (incoming and outgoing NIC limits treated
 * independently, congestion-free core; reading R9).  Path i->j is
 * [up(i), pair(i,j), down(j)]; a capacity of 0 means uncapped (not on the
 * path), < 0 means the link is down.  Nodes with the same site id (or i == j)
 * exchange data in zero time.  Capacities are constant over the batch. */
typedef struct {
  int32_t n_nodes;
  const int64_t *nic_up;    /* [n_nodes] egress cap, bytes/s */
  const int64_t *nic_down;  /* [n_nodes] ingress cap, bytes/s */
  const int64_t *bw;        /* [n_nodes*n_nodes] pair-path caps (row = src) or NULL */
  const int32_t *site;      /* [n_nodes] co-location ids or NULL */
} mlf_net;

/* One batch U: the pushes accumulated since the last plan.
 * node = worker node, bytes = sz(g), version = v(g) (the model version the
 * update was computed from), t_avail_ns = when the update is ready,
 * norm = ||u|| as passed to push(server, update, update_norm) (Table 1). */
typedef struct {
  int32_t n;
  const int32_t *node;
  const int64_t *bytes;
  const int64_t *version;
  const int64_t *t_avail_ns;
  const double *norm;
} mlf_batch;

typedef struct {
  /* parameter-server shards (App. B.2): component j of every update goes to
   * server[j]; component sizes are proportional to shard_weight (NULL = equal):
   * comp_j = floor(B*cum_{j+1}/W) - floor(B*cum_j/W). */
  int32_t n_servers;
  const int32_t *server;
  const int64_t *shard_weight;
  /* pre-assigned aggregators (R13): group i uses agg[i-1] */
  int32_t k;
  const int32_t *agg;
  /* replica: 0 = none, else one node per shard, plus k_r
   * separate replica aggregators */
  int32_t n_replicas;
  const int32_t *replica;
  int32_t k_r;
  const int32_t *replica_agg;
  /* model version after the previous batch and delay bound (Table 1) */
  int64_t v_init;
  int32_t tau_max;
  /* Div_max (Table 1) >= 0, may be +inf; momentum gamma in [0,1) and
   * ||h0|| for the Eq. 9/12 bound (gamma = 0 on the hot path, R15) */
  double div_max, gamma, hist_norm;
  /* replica items punted by the previous batch, in order */
  int32_t n_carried;
  const int32_t *carried_node;
  const int64_t *carried_bytes;
  const double *carried_norm;
  /* 0 = mirror (R16: the frozen prefix is rounded up to a server-commit boundary and the
   * replica receives w there); 1 = replica trees (NEXT-2: the replica applies
   * the frozen replica commits — its own Alg. 3 grouping — and exactly the frozen prefix
   * is frozen, the rest punted) */
  int32_t replica_mode;
  /* 0 = asynchronous SGD (Alg. 2 ordering, deadlines, drops).  1 = synchronous SGD/PS
   * (MLfabric-S: "update ordering does not apply ... aggregation here starts
   * with a list of updates"): O(U) = the batch in submission order, nothing dropped, Alg. 3
   * over that list; one model version per batch (R22).  Also the AllReduce realisation
   * (P:1297-1308): push every update to the (sharded) root with a sync plan, then get. */
  int32_t sync_mode;
} mlf_plan_params;

/* Plan outputs.  All arrays are caller-allocated; `capacity` is their length
 * and must be >= batch n + n_carried, else MLF_E_CAPACITY. */
typedef struct {
  int32_t capacity;
  int32_t n_commit;          /* |O(U)| */
  int32_t *order;            /* [n_commit] batch indices in commit order O(U) (Alg. 2) */
  uint8_t *drop_reason;      /* [n] 0 kept, 1 expired (dl(g) < position), 2 look-ahead drop (Alg. 2 line 10) */
  int32_t *group;            /* [n] 0 direct to server, i >= 1 aggregated in group i (at agg[i-1]), -1 dropped */
  int32_t n_direct;          /* n* of Alg. 3: the first n_direct updates of O(U) go direct */
  int32_t n_groups;
  int32_t *group_node;       /* [n_groups] aggregator node of group i+1 */
  int32_t n_server_commits;  /* commits at the server: n_direct singles, then one per group */
  int32_t *commit_first;     /* [n_server_commits] first position in order[] */
  int32_t *commit_count;     /* [n_server_commits] members (runs over order[]) */
  int64_t *commit_t_ns;      /* [n_server_commits] model commit times (R7), informational */
  int32_t replica_frozen;    /* items of carried ++ order covered by this batch's replica write */
  int32_t replica_boundary_commit; /* mirror point (R16): backup <- w after this many server
                                      commits; 0 = the pre-batch w; -1 = no replica write */
  int32_t n_punted;
  int32_t *punted;           /* [n_punted] indices into carried ++ order, carried to the next batch */
  uint8_t delayed_last;      /* 1 if the last server commit was delayed to meet Div_max (§5.3) */
  int64_t t_total_ns;        /* model time of the last server commit */
  /* the frozen replica commits of the tentative replica plan (Alg. 3 toward the replica on
   * the network after the server plan): runs over carried ++ order */
  int32_t n_replica_commits;
  int32_t *replica_commit_first;   /* [n_replica_commits] (capacity n + n_carried) */
  int32_t *replica_commit_count;
  int32_t *replica_commit_group;   /* 0 direct to the replica, i >= 1 via replica_agg[i-1] */
  int64_t replica_bytes;           /* bytes those commits deliver to the replica nodes */
  uint8_t sync_mode;               /* copied from the params: the executor advances the version by
                                      1 per batch in sync mode, by n_commit otherwise (R2, R22) */
} mlf_plan_out;

/* Alg. 2 -> Alg. 3 -> §5.3 on one batch.  Pure; may run concurrently. */
mlf_status mlf_plan(const mlf_net *net, const mlf_batch *batch,
                    const mlf_plan_params *params, mlf_plan_out *out);

/* ---------------------------------------------------------------------
 * Model distribution trees for pulls (NEXT-4, App. B.3): "for a
 * batch of requests, k° distributors are earmarked.  Mapping of workers to
 * distributors is done using a variant of alg. 3 ... we first transfer the model
 * from the server to the k°-th distributor and then proceed backwards.  The
 * workers in the first group receive the model directly from the server."
 *
 * Reading (R23-R25): Alg. 3 on the time-reversed problem — the network
 * transposed (up <-> down caps, pair (i, j) <-> (j, i)), every request an "update"
 * of model_bytes from its node available at 0, ordered by Alg. 1's SJF (no
 * deadlines); the plan's schedule mirrored by t -> T - t is a feasible real
 * schedule (capacities are constant within a batch, R9). */
typedef struct {
  int32_t n_servers;
  const int32_t *server;           /* [n_servers] shard nodes */
  const int64_t *shard_weight;     /* [n_servers] component weights (App. B.2); NULL = equal */
  int32_t k;                       /* distributors k° */
  const int32_t *distributor;      /* [k] group i -> distributor[i-1] (pre-assigned, as R13) */
  int64_t model_bytes;             /* bytes of one full model (>= 0) */
} mlf_dist_params;

typedef struct {
  int32_t capacity;                /* in: length of the [n] arrays (>= n_requests) */
  int32_t *order;                  /* [n] request indices in SJF order O (R24) */
  int32_t *group;                  /* [n] 0 = direct from the servers, i = via distributor i */
  int32_t n_direct;                /* |group 0| = the chosen n* */
  int32_t n_groups;
  int32_t *group_node;             /* [k] distributor node of group i at [i-1] */
  int64_t t_total_ns;              /* T: every request holds the model by T (model time) */
  int64_t *t_recv_ns;              /* [n] model arrival per request (real time, R25) */
  int64_t *t_start_ns;             /* [n] start of the request's last hop (real time) */
  int64_t *t_dist_ns;              /* [k] model arrival at distributor i (real time) */
} mlf_dist_out;

/* Pure; may run concurrently.  request_node[i] = node of the i-th pull request.
 * Errors: MLF_E_INVALID (null / out-of-range ids, bad weights), MLF_E_CAPACITY
 * (outputs too small), MLF_E_UNSCHEDULABLE (a request's path is down). */
mlf_status mlf_plan_distribution(const mlf_net *net, int32_t n_requests, const int32_t *request_node,
                                 const mlf_dist_params *params, mlf_dist_out *out);

/* ======================================================================
 * Execution (CUDA, one context per process/device; a context is single-threaded)
 * ====================================================================== */

typedef struct {
  int32_t device;              /* CUDA device this context launches on */
  int32_t rank, world;         /* this process serves shard `rank` of `world` PS shards */
  int64_t model_elems;         /* S: full model length in fp32 elements */
  int64_t shard_begin;         /* first element of this rank's shard (multiple of 64) */
  int64_t shard_elems;         /* length of this rank's shard */
  int32_t n_workers;           /* virtual workers; worker w is planner node w */
  mlf_dtype update_dtype;      /* dtype of every update vector */
  float lr;                    /* w <- w - lr * x (R18) */
  float *model_shard;          /* [shard_elems] fp32, on `device` */
  float *backup_shard;         /* [shard_elems] fp32 mirror target of this shard (local or a
                                  mapped peer pointer), or NULL if replication is off */
  void *const *update_slot;    /* [n_workers] full-length update vectors (S elements), each a
                                  device pointer valid on `device` (local or mapped peer) */
  const int32_t *worker_rank;  /* [n_workers] home rank of each worker, or NULL (all local) */
  int32_t n_nodes;             /* planner nodes known to the executor */
  const int32_t *node_rank;    /* [n_nodes] rank hosting each node (aggregators), or NULL (all 0) */
  const int32_t *worker_node;  /* [n_workers] planner node of each worker (the machine/GPU whose NIC
                                  its pushes use), or NULL: worker w is node w */
  int32_t agg_slots;           /* fp32 aggregate buffers per rank for cross-GPU groups (0 = fold groups
                                  inside the commit kernel, no materialised aggregates) */
  float *const *agg_scratch;   /* [world*agg_slots] S-element fp32 buffers valid on `device` */
  void *stream;                /* cudaStream_t (borrowed) */
  /* Momentum (Eq. 2: w <- w + u + gamma (w_t - w_{t-1}), u = -lr * g).  gamma = 0: the
   * hot path above.  gamma in (0,1): the server keeps the history h = w_t - w_{t-1}
   * (history_shard, fp32, shard_elems) and a commit of m updates u_1..u_m applies the
   * aggregate form of m sequential Eq. 2 steps ("consistent to the case with no
   * aggregation"): w += (sum_{j=1..m} g^j) h + sum_i (sum_{j=0..m-i} g^j) u_i,
   * h = g^m h + sum_i g^(m-i) u_i, two weighted sums in one pass (the aggregators'
   * "weighted sum").  backup_history receives h at the mirror boundary.
   * Requires fold mode (agg_slots = 0) and the bulk kernel.  gamma is a double, the same
   * type as mlf_plan_params.gamma (one momentum parameter across the ABI): the weights are
   * computed from it in float64 and each rounded once to fp32 for the kernel (reading R21). */
  double gamma;
  float *history_shard;
  float *backup_history;
  /* Replica trees (NEXT-2; plans with replica_mode = 1): backup_shard is the
   * replica's model shard and mlf_execute applies the plan's frozen replica commits to it
   * (its own grouping, O(U) order).  Updates punted to the next batch are retained: the
   * rank that hosts a punted update copies it into a free slot of its retention pool
   * (slot chosen deterministically, identically on every rank) and the next batch reads it
   * from there as a carried item; the caller must pass the previous plan's punted items, in
   * order, as the next plan's carried items.  retain_slot = [world * n_retain] full-length
   * update buffers (update dtype), local or mapped peer pointers. */
  int32_t replica_mode;
  int32_t n_retain;
  void *const *retain_slot;
  /* Fused get (Table 1 get; the pull of the new model by every GPU): the commit pass
   * also stores each final w tile of this shard into n_bcast full-length fp32 model views
   * (bcast[i] + shard_begin; local or mapped peer pointers) — the all-gather of the new
   * model overlapped tile by tile with the reduce.  Used by the AllReduce realisation
   * (P:1297-1308).  gamma = 0 only; at most 8 destinations. */
  int32_t n_bcast;
  float *const *bcast;
  /* Copy-engine staging (world > 1, fold mode, gamma = 0): operand slices homed on other
   * GPUs are pulled over NVLink by the copy engines into this local buffer, chunk by chunk
   * and double-buffered, while the commit kernel folds the previous chunk from local HBM
   * (copy engines reach a higher NVLink rate than SM peer reads).  NULL / 0 = SM peer reads. */
  void *stage_buf;
  int64_t stage_bytes;
  /* 1: bcast[0] (n_bcast == 1) is an NVLS multicast address bound to every GPU's view (e.g.
   * PyTorch symmetric memory's multicast_ptr): the fused get stores each final tile once
   * with multimem.st and NVSwitch replicates it, instead of one store per peer view. */
  int32_t bcast_multicast;
  /* registerAsServer(params tau_max, ...) (Table 1): the delay bound this server
   * enforces.  enforce_tau = 1: mlf_execute / mlf_execute_phase reject, with MLF_E_INVALID and
   * before any device work, an asynchronous plan (sync_mode = 0) that commits an update g at
   * 1-based position p of O(U) with (v + p) - v(g) > tau_max, v = the context's version
   * (mlf_version) — "no update is applied with a delay greater than tau_max" (P:933-945,
   * reading R1).  A plan built by mlf_plan with the same tau_max and v_init = v never fails the
   * check; a hand-built or stale plan can.  enforce_tau = 0 (a zero-initialised config): not
   * checked.  Synchronous plans have no delay bound. */
  int32_t enforce_tau;
  int32_t tau_max;
} mlf_config;

typedef struct mlf_ctx mlf_ctx;

/* Validate the configuration and create a context at model version v0. */
mlf_status mlf_init(const mlf_config *cfg, int64_t v0, mlf_ctx **out);

/* push(server, update, update_norm) (Table 1): the update vector already
 * sits in the worker's slot; append its descriptor to the current batch.  The
 * slot belongs to the library until the mlf_execute that commits or drops it
 * has completed on-stream (mlf_sync).  Resubmitting a worker already in the
 * batch or still in flight -> MLF_E_STATE.  *index_in_batch (may be NULL)
 * receives the update's batch index. */
mlf_status mlf_submit_update(mlf_ctx *ctx, int32_t worker, int64_t version,
                             int64_t t_avail_ns, double norm, int32_t *index_in_batch);

/* push for n workers in one call (Table 1; the batch of pushes a batching window
 * collects): the same as mlf_submit_update(ctx, worker[i], version[i],
 * t_avail_ns[i], norm[i], NULL) for i = 0..n-1 in that order — the updates take batch indices
 * (current batch size) + i — except that it is all or nothing: every descriptor is checked
 * first and on any error (the codes of mlf_submit_update; a worker twice in `worker` ->
 * MLF_E_STATE) nothing is appended.  worker / version: host arrays of n (borrowed for the
 * call); t_avail_ns / norm: host arrays of n, or NULL for all 0.  n = 0 is a no-op. */
mlf_status mlf_submit_batch(mlf_ctx *ctx, int32_t n, const int32_t *worker,
                            const int64_t *version, const int64_t *t_avail_ns,
                            const double *norm);

/* Optional: worker `worker`'s update lives in pinned host memory `host_ptr`;
 * mlf_execute copies it to the worker's device slot only if the plan commits
 * it (dropped updates are "dropped at the worker itself", and move
 * no bytes).  NULL unregisters. */
mlf_status mlf_set_update_host(mlf_ctx *ctx, int32_t worker, const void *host_ptr);

/* Optional: pinned host buffer (full model length, fp32) that every mlf_execute fills with
 * this rank's shard of the new model (get), at dst + shard_begin.  With host-resident
 * updates on one GPU, mlf_execute then runs as a pipeline over element chunks: the H2D copy
 * of chunk k+1 of the committed updates, the commit of chunk k and the D2H copy of chunk
 * k-1 overlap (copy engines in both directions + SMs).  NULL unregisters. */
mlf_status mlf_set_pull_host(mlf_ctx *ctx, void *host_dst);

/* Borrow the current batch as planner input (arrays valid until the next
 * submit/execute).  bytes = model_elems * sizeof(dtype), node = worker_node[worker]. */
mlf_status mlf_batch_view(mlf_ctx *ctx, mlf_batch *out);

/* Current model version v_init. */
mlf_status mlf_version(mlf_ctx *ctx, int64_t *version);

/* Execute a plan for the current batch (asynchronously, on cfg.stream).
 * Validates the plan against the batch (MLF_E_INVALID if inconsistent), then
 * launches the fused reduce+scale+apply kernel over this rank's shard: for each
 * server commit c in order, x_c = left fold of its members (O(U) order),
 * w <- w - lr*x_c (two fp32 roundings, R17); backup <- w at the boundary
 * commit (R16).  Version += n_commit; the batch is cleared.
 * With agg_slots > 0 and world > 1 the call is split in two phases (see
 * mlf_execute_phase). */
mlf_status mlf_execute(mlf_ctx *ctx, const mlf_plan_out *plan);

/* Two-phase execution for materialised cross-GPU aggregation trees:
 * phase 1 = tree_reduce of the groups whose aggregator lives on this rank into
 * agg_scratch; phase 2 = the ordered commit reading aggregates (local or peer).
 * The caller must make every rank's phase 1 complete before any rank's phase 2
 * starts (mlf_phase_event + a host barrier).  mlf_execute == phase 1 then 2 when
 * world == 1. */
#define MLF_PHASE_AGGREGATE 1
#define MLF_PHASE_COMMIT 2
mlf_status mlf_execute_phase(mlf_ctx *ctx, const mlf_plan_out *plan, int32_t phase);

/* Wait for the last execute; *device_ms (may be NULL) = CUDA-event time on cfg.stream from the
 * first device operation of that execute to its last.  With host-resident updates on one GPU
 * (the mlf_set_pull_host / mlf_set_update_host pipeline) the H2D copies run on a separate copy
 * stream and may start before the window opens, overlapping the previous batch; device_ms then
 * covers the compute stream only, and end-to-end rates are taken by wall time.  Releases the
 * batch's slots. */
mlf_status mlf_sync(mlf_ctx *ctx, float *device_ms);

/* Slots are released per executed batch as soon as that batch's device work has finished
 * (checked by mlf_submit_update).  mlf_release waits until at most max_batches executed
 * batches are still running and releases the finished ones' slots: a producer with two
 * slot sets calls mlf_release(ctx, 1) before submitting into the set batch b-1 used, so
 * batch b+1 is submitted, planned and (host-resident updates) copied in while batch b
 * still commits.  MLF_E_INVALID if max_batches < 0.  With world > 1 the release is local:
 * peers' kernels may still read this rank's slots, so a producer refills a slot only after
 * every rank has synced the batch that read it (a host barrier, as multigpu.py does). */
mlf_status mlf_release(mlf_ctx *ctx, int32_t max_batches);

/* get(server, model) (Table 1): copy this rank's shard of the latest
 * committed model to dst + shard_begin (device or host memory, dst_is_host)
 * after the last execute; *version = batch-boundary version (R19). */
mlf_status mlf_pull_model(mlf_ctx *ctx, void *dst, int32_t dst_is_host, int64_t *version);

/* Execute a distribution plan (NEXT-4, App. B.3) for n pull requests on the box:
 * request_node[i] is the node of request i (node -> GPU through mlf_config.node_rank),
 * view[j] a full-length fp32 model view on rank j (16-byte aligned; mapped peer
 * pointers), shard[j] / shard_begin[j] / shard_elems[j] rank j's PS shard.  Each GPU's
 * view is written once, by its earliest hop in the plan: a GPU that hosts the
 * distributor of a non-empty group or a direct request gathers every shard
 * (MLF_PHASE_AGGREGATE, "the workers in the first group receive the model directly
 * from the server"); any other requesting GPU copies its distributor's view with TMA
 * bulk copies (MLF_PHASE_COMMIT), after the peers' phase-1 events — the caller puts a
 * host barrier between the phases when world > 1.  *source (may be NULL) = -1 filled
 * from the servers, r >= 0 copied from rank r, -2 not requested.  Call after the
 * execute whose model is being distributed; mlf_sync times it. */
mlf_status mlf_distribute_phase(mlf_ctx *ctx, const mlf_dist_out *plan, int32_t n_requests,
                                const int32_t *request_node, float *const *view, const float *const *shard,
                                const int64_t *shard_begin, const int64_t *shard_elems, int32_t phase,
                                int32_t *source);

/* Counters: kernels this context launched, and bytes it moved host<->device. */
mlf_status mlf_stats(mlf_ctx *ctx, int64_t *kernel_launches, int64_t *h2d_bytes, int64_t *d2h_bytes);

void mlf_destroy(mlf_ctx *ctx);

const char *mlf_last_error(void);

/* ======================================================================
 * Peer memory (one process per GPU; NVLink through NVSwitch)
 * ====================================================================== */
typedef struct {
  uint8_t handle[64];        /* cudaIpcMemHandle_t of the allocation containing the pointer */
  int64_t offset;            /* pointer - allocation base */
} mlf_ipc_handle;

mlf_status mlf_ipc_export(int32_t device, const void *dev_ptr, mlf_ipc_handle *out);
/* Map a peer allocation into this process on `device`; *dev_ptr = base + offset. */
mlf_status mlf_ipc_open(int32_t device, const mlf_ipc_handle *h, void **dev_ptr);
mlf_status mlf_ipc_close(int32_t device, void *dev_ptr, int64_t offset);

/* Cross-process ordering of the two execution phases without a device-idle host
 * barrier: every context owns an interprocess "phase 1 done" event, recorded on
 * its stream at the end of mlf_execute_phase(MLF_PHASE_AGGREGATE).  Before its
 * phase 2 launches a context waits (cudaStreamWaitEvent) on the events opened
 * with mlf_phase_events_open.  The caller must order the calls: every rank's
 * phase-1 call returns (record enqueued) before any rank calls phase 2 — a host
 * barrier between the two calls, which overlaps with the GPUs' phase-1 work. */
typedef struct {
  uint8_t handle[64];        /* cudaIpcEventHandle_t */
} mlf_ipc_event;
mlf_status mlf_phase_event_export(mlf_ctx *ctx, mlf_ipc_event *out);
mlf_status mlf_phase_events_open(mlf_ctx *ctx, int32_t n, const mlf_ipc_event *peer_events);

/* get(server, model) of the whole model on one GPU (Table 1): copy n shards (local
 * or mapped peer fp32 buffers) into dst[begin_i .. begin_i + elems_i).  copy_engine = 0:
 * TMA bulk copies (16 KB chunks through shared memory, all shards in one launch) — the
 * NVLink all-gather; 1: one cudaMemcpyAsync per shard on a copy engine; 2: 128-bit SM
 * peer loads (gather_kernel).  Ragged (non-16-byte) tails go to the copy engine.
 * Completes on `stream`. */
mlf_status mlf_gather(int32_t device, float *dst, int32_t n, const float *const *shard, const int64_t *begin,
                      const int64_t *elems, int32_t copy_engine, void *stream);

/* ======================================================================
 * Test infrastructure kernels (not on the hot path)
 * ====================================================================== */

/* Fill dst[0..n) with elements [elem_offset, elem_offset+n) of the synthgen
 * stream (seed, kind, a, b): kind 1 = update of worker a in iteration b,
 * kind 2 = w0.  variant 0 = "normal", 1 = "exact"; dtype F32 or BF16 (kind 2
 * is always F32).  Same counter-based splitmix64 as synthgen/__init__.py,
 * implemented independently.  Launches on `stream`. */
mlf_status mlf_synth_fill(int32_t device, void *dst, int64_t n, int64_t elem_offset,
                          mlf_dtype dtype, uint64_t seed, int32_t kind, int64_t a, int64_t b,
                          int32_t variant, void *stream);

/* Device copy kernel (HBM / NVLink peer roofline denominators): dst <- src, bytes % 16 == 0. */
mlf_status mlf_copy_kernel(int32_t device, void *dst, const void *src, int64_t bytes, void *stream);
/* The same copy on a copy engine (cudaMemcpyAsync device-to-device; peer pointers allowed). */
mlf_status mlf_copy_engine(int32_t device, void *dst, const void *src, int64_t bytes, void *stream);
/* The same copy with TMA bulk copies only (global -> shared -> global, 16 KB chunks). */
mlf_status mlf_copy_bulk(int32_t device, void *dst, const void *src, int64_t bytes, void *stream);
/* Read-only probe: stream `bytes` of src into shared memory with TMA bulk copies, write nothing
 * (the read end of bench.py's mixed read/write HBM ceiling).  src and bytes 16-byte aligned. */
mlf_status mlf_read_probe(int32_t device, const void *src, int64_t bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MLFABRIC_H */
