/*
 * fastb200.h -- C-ABI of the B200-native FAST All-to-All(v) hot path.
 *
 * Plain pointers and sizes only (no torch types).  All device pointers are
 * caller-owned; every call is stream-ordered on `stream` (a cudaStream_t
 * passed as void*), reentrant, and keeps no hidden global state except the
 * communicator objects returned by fast_comm_create.
 *
 * Return codes mirror the reference's error classes (tiersched
 * model.py:29-34) and CLI exit codes (cli.py:420-433):
 *   FAST_OK (0), FAST_EVALIDATION (2) = ValidationError,
 *   FAST_EINVARIANT (3) = InternalInvariantError, FAST_ECUDA (-1) = a CUDA
 *   runtime error (launch failure / bad pointer).
 * Per-matrix outcomes of batched synthesis are written on the device to
 * bufs->status[b] with the same codes.
 */
#ifndef FASTB200_H
#define FASTB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FAST_OK 0
#define FAST_EVALIDATION 2
#define FAST_EINVARIANT 3
#define FAST_ECUDA (-1)

/* Largest server count the batched synthesis kernels accept (stage
 * permutations are uint8, the sort key packs the raw index in 16 bits). */
#define FAST_MAX_SERVERS 128
#define FAST_MAX_GPUS_PER_SERVER 64

/* One balancing move of a cross tile (replaces tiersched IntraMove,
 * balance.py:37-56; `server`/`for_dst_server` are implied by the tile slot). */
typedef struct {
  int64_t bytes;
  int32_t from_gpu;
  int32_t to_gpu;
} fast_move;

/* Where the auxiliary padding of one NW-corner staircase cell (src, dst)
 * runs out (strip_auxiliary, birkhoff.py:225-252: in decomposition order an
 * edge pays its cell's remaining aux before real bytes).  `stage` is the raw
 * index of the LAST stage that charged aux to the cell, `real` the real bytes
 * that edge carried; raw stages before it that use the cell carry 0 real
 * bytes, raw stages after it the full stage weight; every other edge carries
 * the full weight.  stage = -1: unused slot.  With this table the per-edge
 * stage_bytes [K][n] array (16.5 GB per config-5 batch) need not be written. */
typedef struct {
  int64_t real;
  int32_t stage;
  int16_t src;
  int16_t dst;
} fast_strip_rec;

/* Packed schedules for a batch of B matrices with n servers x m GPUs,
 * G = n*m, T = n*(n-1) cross tiles, S = max(m-1,1) move slots per tile,
 * K = n*n-2n+2 stage capacity (birkhoff.py:188).  All device pointers.
 * Replaces the dataclasses Schedule/BalancePlan/Decomposition/
 * PermutationStage (pipeline.py:34-40, balance.py:59-74,
 * birkhoff.py:29-72). */
typedef struct {
  int64_t *balanced;    /* [B][G][G] cross tiles balanced (= redistribution
                           tables, balance.py:129-136), intra tiles = D */
  int64_t *server;      /* [B][n][n] tile totals; diagonal = S_i */
  int32_t *move_count;  /* [B][T] moves per cross tile */
  fast_move *moves;     /* [B][T][S] moves in emission order */
  int64_t *common_sum;  /* [B] max off-diagonal row/col sum (max_rc) */
  int64_t *aux;         /* [B][n][n] auxiliary padding */
  int32_t *n_raw;       /* [B] raw (pre-strip) stage count */
  int64_t *stage_weight;/* [B][K] raw stage weights in decomposition order */
  uint8_t *stage_perm;  /* [B][K][n] dst server of src u in raw stage k */
  int64_t *stage_bytes; /* [B][K][n] real bytes on edge (u, perm[u]), or NULL
                           (then use `strip`) */
  int32_t *n_stages;    /* [B] stages kept after stripping */
  int32_t *stage_order; /* [B][K] raw index of the k-th stage, ascending */
  int32_t *status;      /* [B] FAST_OK / FAST_EVALIDATION / FAST_EINVARIANT */
  void *workspace;      /* fast_synth_workspace_bytes(B, n) bytes */
  /* optional outputs (NULL = not produced) */
  fast_strip_rec *strip;/* [B][2n+2] aux run-out table (above) */
  uint64_t *tile_mask;  /* [B][T] cells of each balanced cross tile that
                           differ from D: bit p*m+q (m <= 8 only) */
} fast_sched_bufs;

/* Library / ABI version (major*10000 + minor*100 + patch). */
int fast_version(void);

/* Workspace needed by fast_synth_batch / fast_decompose_batch. */
size_t fast_synth_workspace_bytes(int B, int n);

/* synthesize_fast for a batch (replaces tiersched.pipeline.synthesize_fast,
 * pipeline.py:52-59): validation (model.py:86-100), build_balance_plan
 * (balance.py:139-174), reduce_to_server_level (model.py:169-178),
 * decompose_server_matrix (birkhoff.py:269-280), strip_auxiliary
 * (birkhoff.py:225-252), sort_stages_ascending (birkhoff.py:255-266).
 * D: device int64 [B][G][G]; for even m, D and out->balanced must be
 * 16-byte aligned (cudaMalloc'd / torch storage is), else FAST_EVALIDATION. */
int fast_synth_batch(const int64_t *D, int B, int n, int m,
                     const fast_sched_bufs *out, void *stream);

/* fast_synth_batch with timing events: if `events` is non-NULL it points to
 * four cudaEvent_t recorded on `stream` before the balance kernel, after it,
 * after the decompose kernel and after the sort kernel (per-kernel device
 * time for the benchmark's roofline). */
int fast_synth_batch_ev(const int64_t *D, int B, int n, int m,
                        const fast_sched_bufs *out, void *stream,
                        void *const *events);

/* Compact result for shipping a batch to the host (the e2e path): after
 * fast_synth_batch with `tile_mask` set, gather the changed cells of every
 * balanced cross tile (tile order i-major, then bit order) into `vals` and
 * write val_base[b] = first value of matrix b (exclusive prefix, val_base[B]
 * = total).  The host rebuilds `balanced` as D with those cells replaced
 * (10.3 of 64 cells per tile at config 5: 1.5 MB instead of 8.4 MB per
 * matrix).  vals capacity: B*T*m*m.  m <= 8. */
size_t fast_compact_workspace_bytes(int B);
int fast_compact_batch(const fast_sched_bufs *out, int B, int n, int m,
                       int64_t *vals, int64_t *val_base, void *workspace,
                       void *stream);

/* build_balance_plan only (balance.py:139-174): fills balanced, server,
 * move_count, moves, status. */
int fast_balance_batch(const int64_t *D, int B, int n, int m,
                       const fast_sched_bufs *out, void *stream);

/* Decomposition of server-level matrices (birkhoff.py:269-280) with
 * stripping and sorting.  mode FAST_DEC_SERVER: S is a ServerMatrix
 * (diagonal ignored, embedding applied, birkhoff.py:75-108); mode
 * FAST_DEC_DOUBLY_STOCHASTIC: S is already doubly stochastic and is
 * decomposed as-is (decompose, birkhoff.py:140-222; aux = 0). */
#define FAST_DEC_SERVER 0
#define FAST_DEC_DOUBLY_STOCHASTIC 1
int fast_decompose_batch(const int64_t *S, int B, int n, int mode,
                         const fast_sched_bufs *out, void *stream);

/* Stage-level building blocks of the Birkhoff module, standalone
 * (csrc/stages.cu; the batched synthesis fuses them).
 *
 * find_perfect_matching (birkhoff.py:111-137) for B boolean supports
 * [B][n][n] (non-zero = edge): rows in index order, columns scanned in
 * index order, fresh `seen` per root.  row_match[b][u] = matched column,
 * status[b] FAST_EINVARIANT (and row_match -1) when no perfect matching. */
int fast_match_batch(const uint8_t *support, int B, int n, int32_t *row_match,
                     int32_t *status, void *stream);

/* strip_auxiliary (birkhoff.py:225-252, mode bit 1) and/or
 * sort_stages_ascending (birkhoff.py:255-266, mode bit 2) on one stage
 * list of K stages over n servers: weight[K], dst[K][n] (-1 = no edge from
 * that source), bytes[K][n], aux[n][n] (strip only).  real_out[K][n]: the
 * edges' bytes after stripping; order_out[0..n_out): input positions of the
 * resulting stages in output order (kept stages in decomposition order, or
 * sorted by (weight, first edge, position)).  status FAST_EINVARIANT when
 * auxiliary bytes are left unconsumed. */
size_t fast_strip_sort_workspace_bytes(int K, int n);
int fast_strip_sort(const int64_t *weight, const int16_t *dst, const int64_t *bytes,
                    const int64_t *aux, int K, int n, int mode, int32_t *order_out,
                    int64_t *real_out, int32_t *n_out, int32_t *status, void *workspace,
                    void *stream);

/* ------------------------------------------------------------------------
 * Executor: P2P stage execution over NVSwitch (replaces the reference's
 * analytical "executor" simulate_fast, simulate.py:107-193, with real data
 * movement; the paper's transfer engine is PAPER.md:605-619).
 * ------------------------------------------------------------------------ */

/* op phases, in execution-priority order */
#define FAST_PH_BALANCE 0      /* giver -> taker staging (balance.py:77-126) */
#define FAST_PH_DIRECT 1       /* intra tile, or stage send of own bytes     */
#define FAST_PH_FROM_STAGING 2 /* stage send of balanced-in bytes           */
#define FAST_PH_REDIST 3       /* proxy staging -> final GPU (balance.py:210)*/
#define FAST_STAGE_INTRA 255  /* fast_op.stage of an intra-server tile copy */
#define FAST_BUF_SEND 0
#define FAST_BUF_RECV 1
#define FAST_BUF_STAGING 2

/* One byte-range copy executed by `exec_rank` into `dst_rank`'s buffer,
 * moved in chunks of the plan's chunk size.  Ops that land in a peer's
 * staging own `nchunks(len)` flag slots there starting at sig_slot (each
 * chunk publishes its slot with the call's epoch); ops that read staging
 * wait for the producer chunks covering [wait_off, wait_off + len) of the
 * producer op whose slots start at wait_slot (on the executing rank). */
typedef struct {
  int64_t src_off;
  int64_t dst_off;
  int64_t len;
  int64_t wait_off;
  int32_t sig_slot;  /* -1: lands in recv (counted) */
  int32_t wait_slot; /* -1: no dependency */
  int16_t exec_rank;
  int16_t dst_rank;
  uint8_t src_buf;
  uint8_t dst_buf;
  uint8_t phase;
  uint8_t stage; /* position in the ascending stage order
                    (FAST_STAGE_INTRA for intra-server tile copies) */
} fast_op;

/* Flag slots per rank available to one plan (fast_comm flags region). */
#define FAST_MAX_SLOTS 65536

/* Compiled plan buffers (device pointers, caller-owned). */
typedef struct {
  fast_op *ops;          /* [op_capacity] */
  int32_t *n_ops;        /* [1] */
  int64_t *staging_used; /* [G] staging bytes needed per rank */
  int32_t *status;       /* [1] */
  void *workspace;       /* fast_plan_workspace_bytes(n, m) */
  int64_t op_capacity;
} fast_plan;

size_t fast_plan_workspace_bytes(int n, int m);
int64_t fast_plan_op_capacity(int n, int m);

/* Plan compile on the device (one-thread kernel, stream-ordered): D [G][G]
 * (zero diagonal) and the packed schedule of matrix 0 of `sched` ->
 * phase-ordered ops.  send_self (device int64[G] or NULL): bytes of each
 * rank's own segment, kept in place inside its send buffer and left as a
 * gap at its slot of the receive buffer (the all_to_all_single layout on
 * both sides); self bytes are never transferred. */
int fast_plan_compile(const int64_t *D, const int64_t *send_self, int n, int m,
                      const fast_sched_bufs *sched, int64_t recv_capacity,
                      int64_t staging_capacity, int64_t chunk_bytes,
                      const fast_plan *plan, void *stream);

/* fast_plan_compile with flags: FAST_PLAN_COPY_SELF also emits each rank's
 * own segment (send_self bytes) as a local DIRECT op into its recv gap. */
#define FAST_PLAN_COPY_SELF 1
int fast_plan_compile_ex(const int64_t *D, const int64_t *send_self, int n, int m,
                         const fast_sched_bufs *sched, int64_t recv_capacity,
                         int64_t staging_capacity, int64_t chunk_bytes,
                         const fast_plan *plan, int flags, void *stream);

/* Same plan logic on HOST pointers -- validation/inspection only (CPU
 * tests); the executor never calls it.  `order/perm/sbytes` are one
 * matrix's packed stage arrays, K = n*n-2n+2. */
int fast_plan_compile_host(const int64_t *D, const int64_t *send_self, int n,
                           int m, int n_stages,
                           const int32_t *order, const uint8_t *perm,
                           const int64_t *sbytes, int64_t recv_capacity,
                           int64_t staging_capacity, int64_t chunk_bytes,
                           fast_op *ops,
                           int64_t op_capacity, int32_t *n_ops,
                           int64_t *staging_used, void *workspace);

/* Communicator: one process per GPU; each rank owns one symmetric
 * allocation [flags | demand x2 | recv | staging] exported by CUDA IPC. */
typedef struct fast_comm fast_comm;

int fast_comm_create(int rank, int world, int max_gpus_per_row,
                     int64_t recv_bytes, int64_t staging_bytes,
                     fast_comm **out);
/* 64-byte cudaIpcMemHandle_t of this rank's symmetric allocation. */
int fast_comm_ipc_handle(const fast_comm *c, void *handle64);
/* handles: world x 64 bytes gathered from every rank (own entry ignored). */
int fast_comm_open_peers(fast_comm *c, const void *handles);
int fast_comm_destroy(fast_comm *c);
void *fast_comm_recv_ptr(const fast_comm *c);
void *fast_comm_staging_ptr(const fast_comm *c);
/* demand-matrix buffer of call `epoch` (double-buffered by parity; epoch <= 0:
 * the fixed slot holding the latest gathered matrix): G x G int64 with zero
 * diagonal, followed by G int64 self-segment sizes */
int64_t *fast_comm_demand_ptr(const fast_comm *c, int64_t epoch);
int64_t fast_comm_recv_capacity(const fast_comm *c);
int64_t fast_comm_staging_capacity(const fast_comm *c);

/* All-gather of this rank's demand row (int64[world], device; entry `rank`
 * = bytes of its own segment, kept local) into every rank's demand buffer for `epoch` (>= 1, +1 per call): P2P writes + a
 * release counter; returns after the local matrix is complete (on the
 * device, stream-ordered).  Replaces Megatron's count all-gather
 * (PAPER.md:617-619). */
int fast_gather_demand(fast_comm *c, const int64_t *row, int64_t epoch,
                       void *stream);

/* Measured per-phase timeline of one exec on one rank (%globaltimer ns;
 * int64 [FAST_TIMELINE_STRIDE] per rank).  Windows are (first chunk start,
 * last chunk end) over the chunks THIS rank executes; 0 / INT64_MAX-like
 * sentinels (start = -1 as unsigned max) mean "no such chunk".  Mirrors the
 * phase breakdown of the reference's Timeline (simulate.py:38-55). */
#define FAST_TL_START 0        /* exec kernel start (CTA 0) */
#define FAST_TL_BARRIER 1      /* entry barrier passed */
#define FAST_TL_OWN_DONE 3     /* CTA 0 left the chunk loop */
#define FAST_TL_RECV_DONE 4    /* every chunk addressed to this rank landed */
#define FAST_TL_BALANCE 8      /* [8] start, [9] end: balance pushes */
#define FAST_TL_INTRA 10       /* [10] start, [11] end: intra-server tiles */
#define FAST_TL_STAGE0 16      /* [16 + 4k + 0/1] stage k sends (scale-out),
                                  [16 + 4k + 2/3] stage k redistribution */
#define FAST_TIMELINE_STRIDE (16 + 4 * 256)

/* Execute a compiled plan: one persistent kernel per rank (`blocks` CTAs);
 * entry barrier, then producer CTAs run balance pushes, intra copies and
 * stage sends while a byte-proportional set of CTAs forwards redistribution
 * chunks as soon as their producer chunks have landed; chunk_bytes must be
 * the plan's.
 * On return (stream order) the local recv buffer holds the alltoallv
 * result.  timeline_ns (device int64[FAST_TIMELINE_STRIDE] or NULL)
 * receives the measured timeline above. */
int fast_exec(fast_comm *c, const fast_plan *plan, const void *send,
              int64_t epoch, int blocks, int64_t chunk_bytes,
              int64_t *timeline_ns, void *stream); /* epoch 0: device counter */
/* One-GPU group mode (testing the full protocol on a single device): `world`
 * communicators whose symmetric blocks all live on the current device, and
 * one cooperative launch (grid = blocks x world, all CTAs co-resident) that
 * runs every rank's part of the plan.  sends: host array of `world` device
 * pointers.  timeline_ns: world x FAST_TIMELINE_STRIDE int64 or NULL. */
int fast_comm_create_group(int world, int64_t recv_bytes, int64_t staging_bytes,
                           fast_comm **comms);
int fast_exec_group(fast_comm *const *comms, int world, const fast_plan *plan,
                    const void *const *sends, int64_t epoch, int blocks,
                    int64_t chunk_bytes, int64_t *timeline_ns, void *stream);
/* One FAST alltoallv, everything enqueued on `stream` (no host sync):
 * demand all-gather of `counts` (device int64[world], entry `rank` = own
 * segment kept in place), synthesis into `sched` (B = 1), plan compile into
 * `plan`, P2P execution.  The receive buffer (fast_comm_recv_ptr) then holds
 * the all_to_all_single layout with a gap at the self slot.  Every argument
 * of the enqueued launches is call-invariant (the epoch lives on the
 * device), so a call can be captured once in a CUDA graph and replayed.
 * Replaces the paper's all_to_all_FAST runtime call. */
int fast_alltoallv(fast_comm *c, const void *send, const int64_t *counts, int n,
                   int m, const fast_sched_bufs *sched, const fast_plan *plan,
                   int blocks, int64_t chunk_bytes, int64_t *timeline_ns,
                   void *stream);
/* fast_alltoallv runs gather + synthesis + plan inside the exec kernel's
 * CTA 0 (one launch per call) when n <= 6 and this is enabled; the default
 * is the multi-launch path (measured equal or faster on B200, see
 * profiles/README.md). */
int fast_comm_set_fused(fast_comm *c, int enable);
/* Fused MoE pack -> send: while set, the executor
 * reads every SEND byte through a row map instead of a packed send buffer:
 * virtual send row r is row row_src[r] of rows_base (row_bytes each, 16-byte
 * multiple; n_rows virtual rows, n_rows * row_bytes / 16 < 2^32).  The send
 * pointer passed to fast_exec / fast_alltoallv is then ignored for data.
 * Launch arguments are taken at enqueue time; row_src == NULL clears it. */
int fast_comm_set_send_rows(fast_comm *c, const void *rows_base,
                            const int32_t *row_src, int64_t row_bytes,
                            int64_t n_rows);
/* fast_alltoallv also moves each rank's own segment (send_self bytes, kept
 * in place in the send buffer) into the gap at its slot of the receive
 * buffer, as one more local DIRECT op run by the exec CTAs alongside the
 * remote sends (row-mapped if fast_comm_set_send_rows is active): the
 * receive region is then the complete all_to_all_single output.  Off by
 * default (the gap is the caller's). */
int fast_comm_set_copy_self(fast_comm *c, int enable);
/* Programmatic dependent launch on the fast_alltoallv chain (gather ->
 * synthesis -> plan -> exec: each kernel launches while its predecessor
 * runs and waits for its memory with griddepcontrol.wait); on by default. */
int fast_comm_set_pdl(fast_comm *c, int enable);
/* Bytes the executor may read from the send side (the send buffer, or
 * n_rows * row_bytes of a row-mapped send); -1 (default) = unchecked.  Taken
 * at enqueue time.  An op reaching past it makes the exec copy nothing and
 * set status 2 (fast_comm_status). */
int fast_comm_set_send_capacity(fast_comm *c, int64_t bytes);
/* Number of calls issued through fast_alltoallv (the current epoch); callers
 * that drive fast_gather_demand / fast_exec themselves report theirs with
 * fast_comm_set_epoch so both paths share one monotone counter. */
int64_t fast_comm_epoch(const fast_comm *c);
int fast_comm_set_epoch(fast_comm *c, int64_t epoch);

/* Base of `rank`'s symmetric block as mapped in this process (own block for
 * rank == own rank); NULL before fast_comm_open_peers. */
void *fast_comm_peer_ptr(const fast_comm *c, int rank);

/* Diagnostics: the executor's CTA copy loop on raw pointers (either side
 * may be a peer mapping) -- NVLink push/pull characterisation only. */
int fast_debug_copy(void *dst, const void *src, int64_t bytes, int blocks,
                    int64_t chunk, int nc, void *stream);

/* Diagnostics: a copy-engine copy (cudaMemcpyAsync) of the same bytes, for
 * the in-run SM-store vs copy-engine NVLink peak measurement. */
int fast_debug_memcpy(void *dst, const void *src, int64_t bytes, void *stream);

/* Device status word of the last exec on this comm: 0 ok, 2 = the counts
 * overran the send capacity (fast_comm_set_send_capacity), 3 = a wait timed
 * out (peers missing or protocol error).  A non-zero status is sticky and
 * leaves the communicator's counters out of step with its peers: destroy
 * and recreate the communicator on every rank. */
int fast_comm_status(const fast_comm *c, int32_t *status_host);

/* ------------------------------------------------------------------------
 * MoE dispatch front-end (BASELINE config 3).  Absent from the reference
 * (its traffic matrices are inputs); the paper takes them from Megatron's
 * count all-gather.  Expert e lives on rank e (E = G).
 * ------------------------------------------------------------------------ */

/* Deterministic top-2 gating of T tokens: r1 = stream(seed)[t] >> 32,
 * r2 = stream(seed)[T+t] >> 32; e1 = #{thr[i] <= r1}, e2 = #{thr2[e1][i] <= r2}
 * (searchsorted 'right' on integer CDFs; thr2[e] has expert e's mass
 * removed).  topk: int32 [T][2]. */
int fast_moe_gate(int T, uint64_t seed, int E, const uint64_t *thr,
                  const uint64_t *thr2, int32_t *topk, void *stream);

/* Histogram + scan of the T*k routing entries (token order): stable rank of
 * every entry inside its destination segment (pos), counts[E], segment row
 * offsets seg_rows[E] (exclusive prefix) and the demand row in bytes
 * (counts * row_bytes) -- this GPU's row of D.  workspace:
 * fast_moe_route_workspace_bytes(T, k, E) bytes (per-block bases, read by
 * fast_moe_pack). */
size_t fast_moe_route_workspace_bytes(int T, int k, int E);
int fast_moe_route(const int32_t *topk, int T, int k, int E, int64_t row_bytes,
                   int32_t *pos, int64_t *counts, int64_t *seg_rows,
                   int64_t *demand_row, void *workspace, void *stream);

/* fast_moe_route with E experts spread over E / experts_per_rank ranks
 * (rank r hosts experts [r*L, (r+1)*L)): counts / seg_rows are per expert
 * (the send layout is expert-major, hence rank-major), demand_row per rank.
 * topk may come from a real router: ids outside [0, E) are rejected (the
 * demand row is set to -1, so the alltoallv fails validation loudly). */
int fast_moe_route_ex(const int32_t *topk, int T, int k, int E, int experts_per_rank,
                      int64_t row_bytes, int32_t *pos, int64_t *counts, int64_t *seg_rows,
                      int64_t *demand_row, void *workspace, void *stream);

/* Pack: token t's row (row_bytes, 16-byte multiple) is copied to each of its
 * k destination rows of `send` (grouped by destination, stable token
 * order) -- the all_to_all_single send layout, self segment included. */
int fast_moe_pack(const void *tokens, int T, int k, int64_t row_bytes,
                  const int32_t *topk, const int32_t *pos, const void *workspace,
                  int E, const int64_t *seg_rows, void *send, void *stream);

/* Unpack: copy this rank's own segment from `send` into the gap the
 * executor leaves at the self slot of `recv` (fast_plan_compile with
 * send_self); recv then holds the expert input, source-major.  D and
 * self_bytes are the gathered demand matrix / self sizes of the call. */
int fast_moe_unpack_self(const int64_t *D, const int64_t *self_bytes, int G,
                         int rank, const void *send, void *recv, void *stream);

/* Fused pack (with fast_comm_set_send_rows): row_src[row] = t for each of
 * the T*k send rows fast_moe_pack would write, i.e. its destination map
 * inverted; 4 bytes per row instead of row_bytes. */
int fast_moe_rowmap(int T, int k, const int32_t *topk, const int32_t *pos,
                    const void *workspace, int E, const int64_t *seg_rows,
                    int32_t *row_src, void *stream);
/* fast_moe_unpack_self for the row-mapped send: the own segment's rows are
 * read from `tokens` through row_src. */
int fast_moe_unpack_self_rows(const int64_t *D, const int64_t *self_bytes,
                              int G, int rank, const void *tokens,
                              const int32_t *row_src, int64_t row_bytes,
                              void *recv, void *stream);

/* Combine (the second alltoallv of an MoE layer,
 * PAPER.md:120): after the reverse FAST alltoallv (counts = column `rank` of
 * the forward D, self kept local), out[t] = sum_j weights[t][j] * row(t, j)
 * over token t's k experts, bf16 rows, fp32 round-to-nearest multiply/add in
 * j order, bf16 RNE result.  Dfwd: the forward call's gathered D (zero
 * diagonal); expert_out: the expert output in the forward receive layout;
 * comb_recv: the reverse call's receive buffer.  topk/pos/workspace/seg_rows
 * are the forward route's. */
int fast_moe_combine(const void *comb_recv, const void *expert_out,
                     const int64_t *Dfwd, int G, int rank, int T, int k,
                     int64_t row_bytes, const int32_t *topk, const int32_t *pos,
                     const void *workspace, int E, const int64_t *seg_rows,
                     const float *weights, void *out, void *stream);
/* fast_moe_combine with E = G * experts_per_rank experts (fast_moe_route_ex). */
int fast_moe_combine_ex(const void *comb_recv, const void *expert_out,
                        const int64_t *Dfwd, int G, int rank, int T, int k,
                        int64_t row_bytes, const int32_t *topk, const int32_t *pos,
                        const void *workspace, int E, int experts_per_rank,
                        const int64_t *seg_rows, const float *weights, void *out,
                        void *stream);

/* ------------------------------------------------------------------------
 * Analytical cost model, batched.  Replaces the
 * reference's per-schedule Python model:
 *   simulate_fast        simulate.py:107-193  -> t_balance .. total
 *   simulate_spreadout   simulate.py:196-242  -> so_* (server / demand mode)
 *   spreadout_stages     spreadout.py:19-31   -> so_weight
 *   optimal_time, fast_worstcase_time, intra_assumption_holds
 *                        bounds.py:27-76      -> t_optimal, t_worstcase, assumption_ok
 * Same operation order in IEEE double as the reference's Python floats, so
 * every output is bit-identical (tests/test_simulate.py).  Status per
 * matrix: FAST_OK, FAST_EVALIDATION (stages not ascending), FAST_EINVARIANT
 * (stage bytes disagree with the tables, floor violated), or the synthesis
 * status passed in.
 * ---------------------------------------------------------------------- */
typedef struct {
  double scaleup_bw;   /* B1, bytes/s */
  double scaleout_bw;  /* B2, bytes/s */
  double wakeup_delay; /* alpha, s */
} fast_sim_topo;

typedef struct {
  const int64_t *balanced;     /* [B][G][G] cross tiles = redistribution tables,
                                  intra tiles = the original blocks */
  const int64_t *server;       /* [B][n][n] tile totals, diagonal S_i */
  const int64_t *common_sum;   /* [B] max_rc of server */
  const int32_t *move_count;   /* [B][T] balance moves per cross tile */
  const fast_move *moves;      /* [B][T][move_slots] */
  const int32_t *n_stages;     /* [B] sorted stages */
  const int32_t *stage_order;  /* [B][stage_stride] row of the k-th stage */
  const int64_t *stage_weight; /* [B][stage_stride] by row */
  const uint8_t *stage_perm;   /* [B][stage_stride][n] */
  const int64_t *stage_bytes;  /* [B][stage_stride][n]; 0 = no edge,
                                  -1 = an edge carrying 0 bytes */
  const int32_t *status;       /* [B] synthesis status, or NULL */
  const int64_t *demand;       /* [B][G][G] original demand for the spreadout
                                  demand mode, or NULL */
  int move_slots;
  int stage_stride;
} fast_sim_in;

typedef struct {
  double *t_balance;      /* [B] */
  double *t_intra;        /* [B] */
  double *scale_out;      /* [B][stage_stride] */
  double *redistribution; /* [B][stage_stride] */
  double *total;          /* [B] */
  double *t_optimal;      /* [B] */
  double *t_worstcase;    /* [B] */
  int32_t *assumption_ok; /* [B] */
  int64_t *so_weight;     /* [B][n-1] spreadout stage weights */
  double *so_server;      /* [B][n-1] spreadout durations, server-level mode */
  double *so_demand;      /* [B][n-1] demand mode (needs in->demand), or NULL */
  double *so_total;       /* [B][2] server-level / demand-mode totals */
  int32_t *status;        /* [B] */
  void *workspace;        /* fast_sim_workspace_bytes(B, n, m, stage_stride) */
} fast_sim_out;

size_t fast_sim_workspace_bytes(int B, int n, int m, int stage_stride);
int fast_simulate_batch(const fast_sim_in *in, int B, int n, int m,
                        const fast_sim_topo *topo, fast_sim_out *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* FASTB200_H */
