// plan.cuh -- FAST stage plan compile: schedule -> byte-exact copy ops.
//
// The reference defines only byte COUNTS per move / stage (balance.py:177-265,
// simulate.py:107-193).  This file fixes which bytes move (SURVEY.md
// Appendix A), so that every GPU's receive buffer equals a direct alltoallv:
//
//  * send_g holds the segment for destination h at offset sum_{h'<h} D[g,h'];
//    recv_h holds the segment from source g at offset sum_{g'<g} D[g',h].
//  * intra-server tiles (i,i): direct copy g -> h.
//  * balancing: balance_senders (balance.py:77-126) is replayed, each take
//    (g -> h, column q, x bytes) moves the TAIL x bytes of g's segment for
//    (j,q) into h's staging, appended to cell (h,q)'s stream.
//  * lane p of pair (i -> j) streams cells (p,0..m-1) in q order; sorted
//    stage k with edge (i,j,b_k) moves, on lane p, bytes
//    [floor((C_{k-1}+m-1-p)/m), floor((C_k+m-1-p)/m)) of that stream to the
//    proxy GPU p of server j (round-robin apportioning, exact).
//  * bytes whose final GPU q != p land in the proxy's staging and are
//    forwarded to GPU q (redistribution, overlapping later stages).
//
// plan_compile() is __host__ __device__: the executor runs it as a one-thread
// kernel on the device (no host round trip); the host build is exported only
// for CPU-side validation of the plan logic (tests/test_plan.py).
#pragma once
#include <stdint.h>

#include "fastb200.h"

#ifndef FAST_HD
#define FAST_HD __host__ __device__
#endif

namespace fastplan {

// Per-tile take record of the balance replay.
struct Take {
  int64_t x;        // bytes
  int64_t seg_off;  // offset inside the giver's segment for (j, q)
  int64_t stg_off;  // where it lands in the taker's staging
  int32_t g, h, q;  // local giver, taker, column
  int32_t slot;     // first flag slot of its balance op on the taker
};

FAST_HD inline int64_t align16(int64_t x) { return (x + 15) & ~(int64_t)15; }

// Bound on takes per tile: each move drains at most m cells plus one partial.
FAST_HD inline int max_takes(int m) { return m > 1 ? (m - 1) * (m + 1) : 1; }

FAST_HD inline int64_t plan_ws_bytes(int n, int m) {
  const int64_t G = (int64_t)n * m, T = (int64_t)n * (n - 1);
  int64_t b = 0;
  b += 2 * G * G * 8;                    // send_off, recv_off
  b += T * max_takes(m) * sizeof(Take);  // takes
  b += T * 4;                            // take counts
  b += T * m * m * 8;                    // final original-part length per cell
  b += (int64_t)n * n * 8;               // delivered per pair
  b += T * m * 3 * 8;                    // lane cursors (cell q, piece, offset)
  b += G * 8;                            // staging top per rank
  b += G * 8;                            // flag-slot top per rank
  b += (int64_t)m * m * 8 + 64;          // tile scratch
  return align16(b);
}

FAST_HD inline int64_t plan_op_capacity(int n, int m, int K) {
  const int64_t T = (int64_t)n * (n - 1);
  const int64_t takes = T * max_takes(m);
  const int64_t windows = T * (int64_t)m * (K + m + max_takes(m) + 1);
  return takes + (int64_t)n * m * m + 2 * windows + 16;
}

struct PlanIn {
  int n, m, K;               // servers, gpus/server, stage capacity
  const int64_t* D;          // [G][G], zero diagonal
  const int64_t* send_self;  // [G] bytes of g's own segment kept in send_g
                             // (all_to_all_single layout); may be null
  int n_stages;              // sorted kept stages
  const int32_t* order;      // [n_stages] raw stage index
  const uint8_t* perm;       // [K][n]
  const int64_t* sbytes;     // [K][n]
  int64_t recv_cap, staging_cap;
  int64_t op_cap;
  int64_t chunk;             // exec chunk size (flag granularity)
  int copy_self;             // 1: also emit each rank's own segment as a local
                             // DIRECT op (send_self bytes -> its recv gap)
};

struct PlanOut {
  fast_op* ops;              // [op_cap], phase-ordered
  fast_op* scratch;          // [op_cap] bucket area (may alias ops)
  int32_t* n_ops;            // [1]
  int64_t* staging_used;     // [G]
  int32_t* status;           // [1]
  void* ws;                  // plan_ws_bytes(n, m)
};

struct Ws {
  int64_t* send_off;
  int64_t* recv_off;
  Take* takes;
  int32_t* ntakes;
  int64_t* orig_len;
  int64_t* delivered;
  int64_t* cursor;  // [T][m][3]: q, piece index within cell, offset in piece
  int64_t* stg_top;
  int64_t* slot_top;
  int64_t* tbuf;  // [m][m] tile scratch
};

FAST_HD inline Ws carve(void* p, int n, int m) {
  const int64_t G = (int64_t)n * m, T = (int64_t)n * (n - 1);
  char* c = (char*)p;
  Ws w;
  w.send_off = (int64_t*)c; c += G * G * 8;
  w.recv_off = (int64_t*)c; c += G * G * 8;
  w.takes = (Take*)c; c += T * max_takes(m) * sizeof(Take);
  w.ntakes = (int32_t*)c; c += T * 4;
  c = (char*)align16((int64_t)(uintptr_t)c);
  w.orig_len = (int64_t*)c; c += T * m * m * 8;
  w.delivered = (int64_t*)c; c += (int64_t)n * n * 8;
  w.cursor = (int64_t*)c; c += T * m * 3 * 8;
  w.stg_top = (int64_t*)c; c += G * 8;
  w.slot_top = (int64_t*)c; c += G * 8;
  w.tbuf = (int64_t*)c;
  return w;
}

FAST_HD inline int tile_index(int n, int i, int j) { return i * (n - 1) + (j < i ? j : j - 1); }

// Op sink with 4 phase buckets laid out back to back in the output array;
// bucket b occupies [b*cap4, (b+1)*cap4) until the final compaction.
struct Sink {
  fast_op* ops;
  int64_t cap4;
  int64_t cnt[4];
  bool overflow;
  FAST_HD void push(int bucket, const fast_op& o) {
    if (cnt[bucket] >= cap4) { overflow = true; return; }
    ops[bucket * cap4 + cnt[bucket]++] = o;
  }
};

FAST_HD inline fast_op make_op(int phase, int stage, int exec_rank, int src_buf,
                               int64_t src_off, int dst_rank, int dst_buf,
                               int64_t dst_off, int64_t len) {
  fast_op o;
  o.src_off = src_off;
  o.dst_off = dst_off;
  o.len = len;
  o.wait_off = 0;
  o.sig_slot = -1;
  o.wait_slot = -1;
  o.exec_rank = (int16_t)exec_rank;
  o.dst_rank = (int16_t)dst_rank;
  o.src_buf = (uint8_t)src_buf;
  o.dst_buf = (uint8_t)dst_buf;
  o.phase = (uint8_t)phase;
  o.stage = (uint8_t)stage;
  return o;
}

// balance_senders replay with take recording (balance.py:77-126).
FAST_HD inline int replay_balance(int64_t* t /*m*m, modified*/, int m, Take* takes,
                                  int cap) {
  int64_t dev[FAST_MAX_GPUS_PER_SERVER];
  int64_t total = 0;
  for (int p = 0; p < m; ++p) {
    int64_t s = 0;
    for (int q = 0; q < m; ++q) s += t[p * m + q];
    dev[p] = s;
    total += s;
  }
  const int64_t base = total / m, extra = total % m;
  for (int p = 0; p < m; ++p) dev[p] -= base + (p < extra ? 1 : 0);
  int nt = 0;
  for (int guard = 0; guard < m; ++guard) {
    int g = -1, h = -1;
    int64_t dg = 0, dh = 0;
    for (int p = 0; p < m; ++p) {
      if (dev[p] > dg) { dg = dev[p]; g = p; }
      if (dev[p] < dh) { dh = dev[p]; h = p; }
    }
    if (g < 0) return nt;
    if (h < 0) return -1;
    const int64_t chunk = dg < -dh ? dg : -dh;
    int64_t left = chunk;
    while (left > 0) {
      int q = 0;
      int64_t best = t[g * m];
      for (int c = 1; c < m; ++c)
        if (t[g * m + c] > best) { best = t[g * m + c]; q = c; }
      const int64_t take = left < best ? left : best;
      if (take <= 0 || nt >= cap) return -1;
      t[g * m + q] -= take;
      t[h * m + q] += take;
      left -= take;
      Take tk;
      tk.x = take;
      tk.seg_off = t[g * m + q];  // the tail starts where the remainder ends
      tk.stg_off = -1;
      tk.g = g;
      tk.h = h;
      tk.q = q;
      tk.slot = -1;
      takes[nt++] = tk;
    }
    dev[g] -= chunk;
    dev[h] += chunk;
  }
  return -1;
}

// Piece iteration of cell (p, q) of tile (i, j): piece 0 is the original
// part (length orig_len), pieces 1.. are takes with h == p, q == q in order.
FAST_HD inline bool cell_piece(const Ws& w, int tix, int m, int p, int q, int64_t piece,
                               int64_t* len, int* origin, int64_t* seg_off, int* in_staging,
                               int64_t* loc_off, int* slot) {
  *slot = -1;
  if (piece == 0) {
    *len = w.orig_len[(int64_t)tix * m * m + p * m + q];
    *origin = p;
    *seg_off = 0;
    *in_staging = 0;
    *loc_off = 0;
    return true;
  }
  int64_t seen = 0;
  const Take* tk = w.takes + (int64_t)tix * max_takes(m);
  for (int a = 0; a < w.ntakes[tix]; ++a) {
    if (tk[a].h == p && tk[a].q == q) {
      if (++seen == piece) {
        *len = tk[a].x;
        *origin = tk[a].g;
        *seg_off = tk[a].seg_off;
        *in_staging = 1;
        *loc_off = tk[a].stg_off;
        *slot = tk[a].slot;
        return true;
      }
    }
  }
  return false;
}

FAST_HD inline void plan_compile(const PlanIn& in, const PlanOut& out) {
  const int n = in.n, m = in.m;
  const int G = n * m;
  const int T = n * (n - 1);
  Ws w = carve(out.ws, n, m);
  Sink sk;
  sk.ops = out.scratch ? out.scratch : out.ops;
  sk.cap4 = in.op_cap / 4;
  sk.cnt[0] = sk.cnt[1] = sk.cnt[2] = sk.cnt[3] = 0;
  sk.overflow = false;
  int status = FAST_OK;

  if (in.n_stages > 255 || m > FAST_MAX_GPUS_PER_SERVER) status = FAST_EVALIDATION;
  // segment offsets (the self segment, if any, stays in place in send_g)
  for (int g = 0; g < G; ++g) {
    int64_t a = 0;
    for (int h = 0; h < G; ++h) {
      w.send_off[(int64_t)g * G + h] = a;
      a += in.D[(int64_t)g * G + h];
      if (h == g && in.send_self) a += in.send_self[g];
    }
  }
  // recv_h is source-major; with send_self the own segment's slot is left
  // as a gap (filled locally, e.g. by the MoE unpack), so recv_h is laid out
  // exactly like all_to_all_single's output
  for (int h = 0; h < G; ++h) {
    int64_t a = 0;
    for (int g = 0; g < G; ++g) {
      w.recv_off[(int64_t)g * G + h] = a;
      a += in.D[(int64_t)g * G + h];
      if (g == h && in.send_self) a += in.send_self[h];
    }
    if (a > in.recv_cap) status = FAST_EVALIDATION;
  }
  for (int r = 0; r < G; ++r) w.stg_top[r] = 0, w.slot_top[r] = 0;
  const int64_t CH = in.chunk > 0 ? in.chunk : ((int64_t)1 << 20);
  // flag slots of an op that lands in `rank`'s staging (one per chunk)
  auto take_slots = [&](int rank, int64_t len) -> int32_t {
    const int64_t s0 = w.slot_top[rank];
    w.slot_top[rank] = s0 + (len + CH - 1) / CH;
    return (int32_t)s0;
  };
  for (int c = 0; c < n * n; ++c) w.delivered[c] = 0;

  // ---- phase 0: balancing pushes (into the taker's staging) ---------------
  int64_t* tbuf = w.tbuf;
  for (int i = 0; i < n && status == FAST_OK; ++i) {
    for (int j = 0; j < n; ++j) {
      if (i == j) continue;
      const int tix = tile_index(n, i, j);
      for (int p = 0; p < m; ++p)
        for (int q = 0; q < m; ++q)
          tbuf[p * m + q] = in.D[(int64_t)(i * m + p) * G + j * m + q];
      Take* tk = w.takes + (int64_t)tix * max_takes(m);
      const int nt = replay_balance(tbuf, m, tk, max_takes(m));
      if (nt < 0) { status = FAST_EINVARIANT; break; }
      w.ntakes[tix] = nt;
      // remaining original length of every cell: givers shrink, takers keep
      for (int p = 0; p < m; ++p)
        for (int q = 0; q < m; ++q)
          w.orig_len[(int64_t)tix * m * m + p * m + q] = in.D[(int64_t)(i * m + p) * G + j * m + q];
      for (int a = 0; a < nt; ++a) {
        const int gi = i * m + tk[a].g, hi = i * m + tk[a].h, dst = j * m + tk[a].q;
        w.orig_len[(int64_t)tix * m * m + tk[a].g * m + tk[a].q] = tk[a].seg_off;
        tk[a].stg_off = w.stg_top[hi];
        w.stg_top[hi] = align16(w.stg_top[hi] + tk[a].x);
        tk[a].slot = take_slots(hi, tk[a].x);
        fast_op o = make_op(FAST_PH_BALANCE, 0, gi, FAST_BUF_SEND,
                            w.send_off[(int64_t)gi * G + dst] + tk[a].seg_off, hi,
                            FAST_BUF_STAGING, tk[a].stg_off, tk[a].x);
        o.sig_slot = tk[a].slot;
        sk.push(0, o);
      }
      for (int c = 0; c < m * 3; ++c) w.cursor[(int64_t)tix * m * 3 + c] = 0;
    }
  }

  // ---- intra-server tiles: direct copies ----------------------------------
  for (int i = 0; i < n && status == FAST_OK; ++i)
    for (int p = 0; p < m; ++p)
      for (int q = 0; q < m; ++q) {
        const int g = i * m + p, h = i * m + q;
        const int64_t len = g != h ? in.D[(int64_t)g * G + h]
                                   : (in.copy_self && in.send_self ? in.send_self[g] : 0);
        if (len > 0)
          sk.push(1, make_op(FAST_PH_DIRECT, FAST_STAGE_INTRA, g, FAST_BUF_SEND, w.send_off[(int64_t)g * G + h],
                             h, FAST_BUF_RECV, w.recv_off[(int64_t)g * G + h], len));
      }

  // ---- stage windows + redistribution --------------------------------------
  // Within a stage, sends that land in a proxy's staging (and must be
  // forwarded) are emitted before sends that land in their final buffer, so
  // proxies can start forwarding early; bucket 1 = own bytes, 2 = balanced-in
  // bytes (waits for their balance chunks), 3 = redistribution.
  for (int s = 0; s < in.n_stages && status == FAST_OK; ++s) {
    const int k = in.order[s];
    for (int pass = 0; pass < 2 && status == FAST_OK; ++pass) {
      for (int i = 0; i < n && status == FAST_OK; ++i) {
        const int64_t b = in.sbytes[(int64_t)k * n + i];
        if (b <= 0) continue;
        const int j = in.perm[(int64_t)k * n + i];
        const int tix = tile_index(n, i, j);
        const int64_t c0 = w.delivered[i * n + j];
        const int64_t c1 = c0 + b;
        for (int p = 0; p < m; ++p) {
          int64_t want = (c1 + m - 1 - p) / m - (c0 + m - 1 - p) / m;
          int64_t* cur = w.cursor + ((int64_t)tix * m + p) * 3;  // q, piece, off
          int64_t cq = cur[0], cpc = cur[1], coff = cur[2];       // pass-local walk
          const int src_rank = i * m + p, proxy = j * m + p;
          while (want > 0) {
            if (cq >= m) { status = FAST_EINVARIANT; break; }
            int64_t len, seg_off, loc_off;
            int origin, in_stg, slot;
            if (!cell_piece(w, tix, m, p, (int)cq, cpc, &len, &origin, &seg_off, &in_stg,
                            &loc_off, &slot)) {
              cq += 1;  // next cell of the lane stream
              cpc = 0;
              coff = 0;
              continue;
            }
            const int64_t avail = len - coff;
            if (avail <= 0) { cpc += 1; coff = 0; continue; }
            const int64_t x = want < avail ? want : avail;
            const int q = (int)cq;
            const bool staged = q != p;
            if (staged == (pass == 0)) {
              const int fin = j * m + q, orig = i * m + origin;
              const int64_t src_off = in_stg ? loc_off + coff
                                             : w.send_off[(int64_t)src_rank * G + fin] + coff;
              const int64_t fin_off = w.recv_off[(int64_t)orig * G + fin] + seg_off + coff;
              const int bucket = in_stg ? 2 : 1;
              const int ph = in_stg ? FAST_PH_FROM_STAGING : FAST_PH_DIRECT;
              const int sbuf = in_stg ? FAST_BUF_STAGING : FAST_BUF_SEND;
              fast_op o;
              if (!staged) {
                o = make_op(ph, s, src_rank, sbuf, src_off, proxy, FAST_BUF_RECV, fin_off, x);
              } else {
                const int64_t stg = w.stg_top[proxy];
                w.stg_top[proxy] = align16(stg + x);
                o = make_op(ph, s, src_rank, sbuf, src_off, proxy, FAST_BUF_STAGING, stg, x);
                o.sig_slot = take_slots(proxy, x);
                fast_op r = make_op(FAST_PH_REDIST, s, proxy, FAST_BUF_STAGING, stg, fin,
                                    FAST_BUF_RECV, fin_off, x);
                r.wait_slot = o.sig_slot;
                r.wait_off = 0;
                sk.push(3, r);
              }
              if (in_stg) {
                o.wait_slot = slot;  // the balance op that brought these bytes
                o.wait_off = coff;
              }
              sk.push(bucket, o);
            }
            coff += x;
            want -= x;
          }
          if (pass == 1) {  // commit the walk after the second pass
            cur[0] = cq;
            cur[1] = cpc;
            cur[2] = coff;
          }
        }
        if (pass == 1) w.delivered[i * n + j] = c1;
      }
    }
  }
  // every pair fully delivered (simulate.py:127-142)
  for (int i = 0; i < n && status == FAST_OK; ++i)
    for (int j = 0; j < n; ++j) {
      if (i == j) continue;
      int64_t tot = 0;
      for (int p = 0; p < m; ++p)
        for (int q = 0; q < m; ++q) tot += in.D[(int64_t)(i * m + p) * G + j * m + q];
      if (tot != w.delivered[i * n + j]) status = FAST_EINVARIANT;
    }
  for (int r = 0; r < G; ++r) {
    out.staging_used[r] = w.stg_top[r];
    if (w.stg_top[r] > in.staging_cap && status == FAST_OK) status = FAST_EVALIDATION;
    if (w.slot_top[r] > FAST_MAX_SLOTS && status == FAST_OK) status = FAST_EVALIDATION;
  }
  if (sk.overflow && status == FAST_OK) status = FAST_EINVARIANT;
  // compact the buckets: [balance][direct][from staging][redistribution]
  int64_t at = 0;
  for (int bk = 0; bk < 4; ++bk)
    for (int64_t x = 0; x < sk.cnt[bk]; ++x) {
      const fast_op o = sk.ops[bk * sk.cap4 + x];  // forward copy: at <= source index
      out.ops[at++] = o;
    }
  *out.n_ops = status == FAST_OK ? (int32_t)at : 0;
  *out.status = status;
  (void)T;
}

}  // namespace fastplan
