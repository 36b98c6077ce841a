/*
 * fastb200.h -- C-ABI of the B200-native FAST All-to-All(v) hot path.
 *
 * Plain pointers and sizes only (no torch types).  All device pointers are
 * caller-owned; every call is stream-ordered on `stream` (a cudaStream_t
 * passed as void*), reentrant, and keeps no hidden global state except the
 * communicator objects returned by fast_comm_init.
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
  int64_t *stage_bytes; /* [B][K][n] real bytes on edge (u, perm[u]) */
  int32_t *n_stages;    /* [B] stages kept after stripping */
  int32_t *stage_order; /* [B][K] raw index of the k-th stage, ascending */
  int32_t *status;      /* [B] FAST_OK / FAST_EVALIDATION / FAST_EINVARIANT */
  void *workspace;      /* fast_synth_workspace_bytes(B, n) bytes */
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
 * D: device int64 [B][G][G]. */
int fast_synth_batch(const int64_t *D, int B, int n, int m,
                     const fast_sched_bufs *out, void *stream);

/* fast_synth_batch with timing events: if `events` is non-NULL it points to
 * four cudaEvent_t recorded on `stream` before the balance kernel, after it,
 * after the decompose kernel and after the sort kernel (per-kernel device
 * time for the benchmark's roofline). */
int fast_synth_batch_ev(const int64_t *D, int B, int n, int m,
                        const fast_sched_bufs *out, void *stream,
                        void *const *events);

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

#ifdef __cplusplus
}
#endif
#endif /* FASTB200_H */
