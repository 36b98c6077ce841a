/*
 * fast_oracle.c -- CPU ORACLE (test infrastructure only).
 *
 * This file is the checker for the B200 FAST schedule-synthesis path.  It is
 * a plain-C restatement of the reference `tiersched` scheduler
 * (/root/reference/pkg/src/tiersched, pure Python).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it; the
 * product path (paper_2505_09764_b200) never links or calls it.
 *
 * Parity of this restatement is pinned against the reference itself: the
 * committed golden fixtures in tests/golden/ were produced by importing
 * tiersched (tests/golden/make_golden.py) and tests/test_oracle.py checks
 * this oracle against every one of them (canonical-JSON byte equality).
 *
 * Each function cites the reference lines it follows.  It deliberately keeps
 * the reference's control structure (recursive Kuhn DFS with a shared `seen`
 * array, greedy list-sorted balancing, sequential aux charging, stable sort)
 * so that it checks the GPU kernels' different formulation (bitset DFS with an
 * explicit stack, interval-overlap embedding, fused strip) independently.
 *
 * Packed output layout (identical to the GPU's, see include/fastb200.h):
 *   balanced  int64[G*G]   cross tiles balanced (== redistribution tables),
 *                          intra tiles copied from D
 *   server    int64[n*n]   tile totals (diagonal = S_i)
 *   move_count int32[T]    T = n(n-1) cross tiles in (i,j) row-major order
 *   moves     {int64 bytes; int32 from; int32 to}[T][max(m-1,1)]
 *   common    int64        max off-diagonal row/column sum
 *   aux       int64[n*n]
 *   n_raw     int32        raw (pre-strip) stage count
 *   sweight   int64[K]     raw stage weights, K = n*n-2n+2
 *   sperm     uint8[K*n]   raw stage permutation: dst server of src u
 *   sbytes    int64[K*n]   real bytes of edge (u, sperm[u]) after stripping
 *   n_stages  int32        kept (non-empty) stages
 *   order     int32[K]     raw index of the k-th stage in ascending order
 * Return value: 0 ok, 2 validation error, 3 internal invariant broken
 * (ValidationError / InternalInvariantError, model.py:29-34).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int64_t bytes;
    int32_t from_gpu;
    int32_t to_gpu;
} fo_move;

#define FO_OK 0
#define FO_EVALIDATION 2
#define FO_EINVARIANT 3
#define FO_MAX_SAFE_TOTAL (((int64_t)1) << 62) /* model.py:26 */

/* ------------------------------------------------------------------------ */
/* Phase 1: balance_senders (balance.py:77-126), one cross tile.            */
/* tile: m x m, row stride `ld`.  Returns number of moves written.           */
static int fo_balance_senders(int64_t *tile, int ld, int m, fo_move *moves)
{
    int64_t rows[64], target[64], dev[64];
    int64_t total = 0;
    for (int p = 0; p < m; p++) {
        int64_t s = 0;
        for (int q = 0; q < m; q++) s += tile[p * ld + q];
        rows[p] = s;
        total += s;
    }
    int64_t base = total / m, extra = total % m; /* divmod, total >= 0 */
    for (int p = 0; p < m; p++) {
        target[p] = base + (p < extra ? 1 : 0);
        dev[p] = rows[p] - target[p];
    }
    /* over/under lists re-sorted every iteration by (-dev, g) / (dev, g):
     * over[0] is the largest positive deviation, lowest index on ties;
     * under[0] the most negative deviation, lowest index on ties. */
    int nmoves = 0;
    for (;;) {
        int g = -1, h = -1;
        for (int p = 0; p < m; p++) {
            if (dev[p] > 0 && (g < 0 || dev[p] > dev[g])) g = p;
            if (dev[p] < 0 && (h < 0 || dev[p] < dev[h])) h = p;
        }
        if (g < 0) break;
        int64_t chunk = dev[g] < -dev[h] ? dev[g] : -dev[h];
        int64_t left = chunk;
        while (left > 0) {
            /* q = np.argmax(tiled[g]) -- first maximum */
            int q = 0;
            for (int c = 1; c < m; c++)
                if (tile[g * ld + c] > tile[g * ld + q]) q = c;
            int64_t take = left < tile[g * ld + q] ? left : tile[g * ld + q];
            tile[g * ld + q] -= take;
            tile[h * ld + q] += take;
            left -= take;
        }
        dev[g] -= chunk;
        dev[h] += chunk;
        moves[nmoves].bytes = chunk;
        moves[nmoves].from_gpu = g;
        moves[nmoves].to_gpu = h;
        nmoves++;
    }
    return nmoves;
}

/* build_balance_plan (balance.py:139-174) + reduce_to_server_level
 * (model.py:169-178).  D is validated first like DemandMatrix
 * (model.py:86-100). */
int fo_balance(int n, int m, const int64_t *D, int64_t *balanced,
               int64_t *server, int32_t *move_count, fo_move *moves)
{
    const int G = n * m;
    const int slots = m > 1 ? m - 1 : 1;
    if (n < 2 || m < 1 || m > 64) return FO_EVALIDATION;
    /* DemandMatrix validation: non-negative, zero diagonal, total < 2^62. */
    int64_t total = 0;
    for (int g = 0; g < G; g++) {
        if (D[(int64_t)g * G + g] != 0) return FO_EVALIDATION;
        for (int h = 0; h < G; h++) {
            int64_t v = D[(int64_t)g * G + h];
            if (v < 0) return FO_EVALIDATION;
            if (v >= FO_MAX_SAFE_TOTAL - total) return FO_EVALIDATION;
            total += v;
        }
    }
    memcpy(balanced, D, sizeof(int64_t) * (size_t)G * G);
    int t = 0;
    for (int i = 0; i < n; i++) {
        for (int j = 0; j < n; j++) {
            int64_t *blk = balanced + (int64_t)(i * m) * G + j * m;
            int64_t before = 0;
            for (int p = 0; p < m; p++)
                for (int q = 0; q < m; q++) before += blk[(int64_t)p * G + q];
            server[i * n + j] = before;
            if (i == j) continue;
            int nm = fo_balance_senders(blk, G, m, moves + (size_t)t * slots);
            if (nm > slots) return FO_EINVARIANT;
            move_count[t] = nm;
            /* merge_peer (balance.py:129-136): row sums differ by <= 1 */
            int64_t lo = INT64_MAX, hi = INT64_MIN, after = 0;
            for (int p = 0; p < m; p++) {
                int64_t s = 0;
                for (int q = 0; q < m; q++) s += blk[(int64_t)p * G + q];
                if (s < lo) lo = s;
                if (s > hi) hi = s;
                after += s;
            }
            if (hi - lo > 1) return FO_EVALIDATION;
            if (after != before) return FO_EINVARIANT; /* balance.py:157-163 */
            t++;
        }
    }
    return FO_OK;
}

/* ------------------------------------------------------------------------ */
/* Phase 2: embed_doubly_stochastic (birkhoff.py:75-108), northwest corner. */
static int fo_embed(int n, const int64_t *S, int64_t *embedded, int64_t *aux,
                    int64_t *common_out)
{
    int64_t *rowdef = (int64_t *)malloc(sizeof(int64_t) * n);
    int64_t *coldef = (int64_t *)malloc(sizeof(int64_t) * n);
    int64_t common = 0;
    for (int i = 0; i < n; i++) {
        int64_t r = 0, c = 0;
        for (int j = 0; j < n; j++) {
            if (i == j) continue;
            r += S[i * n + j];
            c += S[j * n + i];
        }
        rowdef[i] = r;
        coldef[i] = c;
        if (r > common) common = r;
        if (c > common) common = c;
    }
    for (int i = 0; i < n; i++) {
        for (int j = 0; j < n; j++)
            embedded[i * n + j] = (i == j) ? 0 : S[i * n + j];
        rowdef[i] = common - rowdef[i];
        coldef[i] = common - coldef[i];
    }
    int j = 0;
    for (int i = 0; i < n; i++) {
        int64_t need = rowdef[i];
        while (need > 0) {
            if (j >= n) { free(rowdef); free(coldef); return FO_EINVARIANT; }
            int64_t grant = need < coldef[j] ? need : coldef[j];
            if (grant > 0) {
                embedded[i * n + j] += grant;
                coldef[j] -= grant;
                need -= grant;
            }
            if (coldef[j] == 0) j++;
        }
    }
    int st = FO_OK;
    for (int a = 0; a < n && st == FO_OK; a++) {
        int64_t r = 0, c = 0;
        for (int b = 0; b < n; b++) {
            r += embedded[a * n + b];
            c += embedded[b * n + a];
        }
        if (r != common || c != common) st = FO_EINVARIANT; /* :102-106 */
    }
    for (int a = 0; a < n; a++)
        for (int b = 0; b < n; b++)
            aux[a * n + b] = embedded[a * n + b] - (a == b ? 0 : S[a * n + b]);
    *common_out = common;
    free(rowdef);
    free(coldef);
    return st;
}

/* decompose (birkhoff.py:140-222): recursive Kuhn augmentation. */
typedef struct {
    int n;
    int64_t *work;
    int *row_match, *col_match;
    unsigned char *seen;
} fo_dec;

/* DFS work counters (measurement only: bench.py reports the GPU kernel's
 * cycles per DFS step against them).  One step = one column newly marked
 * seen, i.e. one iteration of the GPU search loop. */
static int64_t fo_steps, fo_searches;
int64_t fo_dfs_counters(int64_t *searches, int reset)
{
    int64_t s = fo_steps;
    if (searches) *searches = fo_searches;
    if (reset) fo_steps = fo_searches = 0;
    return s;
}

static int fo_augment(fo_dec *d, int u) /* birkhoff.py:172-180 */
{
    for (int v = 0; v < d->n; v++) {
        if (d->work[u * d->n + v] > 0 && !d->seen[v]) {
            d->seen[v] = 1;
            fo_steps++;
            if (d->col_match[v] < 0 || fo_augment(d, d->col_match[v])) {
                d->col_match[v] = u;
                d->row_match[u] = v;
                return 1;
            }
        }
    }
    return 0;
}

/* strip_auxiliary (birkhoff.py:225-252) is applied in decomposition order;
 * sort_stages_ascending (birkhoff.py:255-266) is a stable sort on
 * (weight, first-edge (src, dst)). */
typedef struct {
    int64_t w;
    int src0, dst0, idx;
} fo_key;

static int fo_key_cmp(const void *a, const void *b)
{
    const fo_key *x = (const fo_key *)a, *y = (const fo_key *)b;
    if (x->w != y->w) return x->w < y->w ? -1 : 1;
    if (x->src0 != y->src0) return x->src0 < y->src0 ? -1 : 1;
    if (x->dst0 != y->dst0) return x->dst0 < y->dst0 ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx); /* stability */
}

/* decompose_server_matrix (birkhoff.py:269-280) followed by the pipeline's
 * strip + sort (pipeline.py:52-59). */
int fo_decompose_server(int n, const int64_t *S, int64_t *common_out,
                        int64_t *aux, int32_t *n_raw, int64_t *sweight,
                        uint8_t *sperm, int64_t *sbytes, int32_t *n_stages,
                        int32_t *order)
{
    if (n < 2 || n > 255) return FO_EVALIDATION;
    const int K = n * n - 2 * n + 2;
    int64_t *emb = (int64_t *)malloc(sizeof(int64_t) * n * n);
    int64_t common = 0;
    int st = fo_embed(n, S, emb, aux, &common);
    *common_out = common;
    *n_raw = 0;
    *n_stages = 0;
    if (st != FO_OK || common == 0) { free(emb); return st; }

    fo_dec d;
    d.n = n;
    d.work = emb;
    d.row_match = (int *)malloc(sizeof(int) * n);
    d.col_match = (int *)malloc(sizeof(int) * n);
    d.seen = (unsigned char *)malloc(n);
    int *freed = (int *)malloc(sizeof(int) * n);
    int64_t *aux_left = (int64_t *)malloc(sizeof(int64_t) * n * n);
    memcpy(aux_left, aux, sizeof(int64_t) * n * n);
    for (int u = 0; u < n; u++) d.row_match[u] = d.col_match[u] = -1;

    for (int u = 0; u < n && st == FO_OK; u++) {
        memset(d.seen, 0, n);
        fo_searches++;
        if (!fo_augment(&d, u)) st = FO_EINVARIANT;
    }
    int64_t remaining = common;
    int k = 0;
    while (st == FO_OK && remaining > 0) {
        if (k >= K) { st = FO_EINVARIANT; break; }
        int64_t weight = INT64_MAX;
        for (int u = 0; u < n; u++) {
            int64_t x = d.work[u * n + d.row_match[u]];
            if (x < weight) weight = x;
        }
        if (weight <= 0) { st = FO_EINVARIANT; break; }
        sweight[k] = weight;
        remaining -= weight;
        int nf = 0;
        for (int u = 0; u < n; u++) {
            int v = d.row_match[u];
            sperm[(int64_t)k * n + u] = (uint8_t)v;
            /* strip: this edge pays its cell's auxiliary bytes first */
            int64_t charged = aux_left[u * n + v] < weight ? aux_left[u * n + v]
                                                           : weight;
            aux_left[u * n + v] -= charged;
            sbytes[(int64_t)k * n + u] = weight - charged;
            d.work[u * n + v] -= weight;
            if (d.work[u * n + v] == 0 && remaining > 0) freed[nf++] = u;
        }
        k++;
        for (int f = 0; f < nf; f++) {
            int u = freed[f], v = d.row_match[u];
            if (d.col_match[v] == u) d.col_match[v] = -1;
            d.row_match[u] = -1;
        }
        for (int f = 0; f < nf && st == FO_OK; f++) {
            int u = freed[f];
            if (d.row_match[u] < 0) {
                memset(d.seen, 0, n);
                fo_searches++;
                if (!fo_augment(&d, u)) st = FO_EINVARIANT;
            }
        }
    }
    *n_raw = k;
    if (st == FO_OK) {
        for (int c = 0; c < n * n; c++)
            if (d.work[c] != 0 || aux_left[c] != 0) st = FO_EINVARIANT;
    }
    if (st == FO_OK) {
        int64_t tw = 0;
        for (int s = 0; s < k; s++) tw += sweight[s];
        if (tw != common) st = FO_EINVARIANT; /* birkhoff.py:273-277 */
    }
    if (st == FO_OK) {
        fo_key *keys = (fo_key *)malloc(sizeof(fo_key) * (k > 0 ? k : 1));
        int kept = 0;
        for (int s = 0; s < k; s++) {
            int src0 = -1;
            for (int u = 0; u < n; u++)
                if (sbytes[(int64_t)s * n + u] > 0) { src0 = u; break; }
            if (src0 < 0) continue; /* empty stages disappear */
            keys[kept].w = sweight[s];
            keys[kept].src0 = src0;
            keys[kept].dst0 = sperm[(int64_t)s * n + src0];
            keys[kept].idx = s;
            kept++;
        }
        qsort(keys, kept, sizeof(fo_key), fo_key_cmp);
        for (int s = 0; s < kept; s++) order[s] = keys[s].idx;
        *n_stages = kept;
        free(keys);
    }
    free(d.row_match);
    free(d.col_match);
    free(d.seen);
    free(freed);
    free(aux_left);
    free(emb);
    return st;
}

/* synthesize_fast (pipeline.py:52-59): balance, reduce, decompose, strip,
 * sort -- for one demand matrix. */
int fo_synthesize(int n, int m, const int64_t *D, int64_t *balanced,
                  int64_t *server, int32_t *move_count, fo_move *moves,
                  int64_t *common, int64_t *aux, int32_t *n_raw,
                  int64_t *sweight, uint8_t *sperm, int64_t *sbytes,
                  int32_t *n_stages, int32_t *order)
{
    int st = fo_balance(n, m, D, balanced, server, move_count, moves);
    if (st != FO_OK) return st;
    return fo_decompose_server(n, server, common, aux, n_raw, sweight, sperm,
                               sbytes, n_stages, order);
}

/* Batched driver for the CPU baseline: B matrices, contiguous packed
 * buffers, stride per matrix as in the GPU layout.  status[b] per matrix. */
int fo_synthesize_batch(int B, int n, int m, const int64_t *D,
                        int64_t *balanced, int64_t *server,
                        int32_t *move_count, fo_move *moves, int64_t *common,
                        int64_t *aux, int32_t *n_raw, int64_t *sweight,
                        uint8_t *sperm, int64_t *sbytes, int32_t *n_stages,
                        int32_t *order, int32_t *status)
{
    const int64_t G = (int64_t)n * m, T = (int64_t)n * (n - 1);
    const int64_t slots = m > 1 ? m - 1 : 1, K = (int64_t)n * n - 2 * n + 2;
    int worst = FO_OK;
    for (int b = 0; b < B; b++) {
        int st = fo_synthesize(
            n, m, D + b * G * G, balanced + b * G * G, server + b * n * n,
            move_count + b * T, moves + b * T * slots, common + b,
            aux + b * n * n, n_raw + b, sweight + b * K, sperm + b * K * n,
            sbytes + b * K * n, n_stages + b, order + b * K);
        status[b] = st;
        if (st > worst) worst = st;
    }
    return worst;
}
