"""Schedule containers, the packed device layout, and canonical JSON.

The dataclasses mirror tiersched's (balance.py:37-74, birkhoff.py:29-72,
pipeline.py:34-40) so that ``schedule_to_json`` of a GPU-synthesized schedule
is byte-identical to the reference's (pipeline.py:72-145).  ``PackedSchedule``
is the host view of one matrix of ``fast_sched_bufs`` (include/fastb200.h);
``to_schedule`` rebuilds the dataclasses from it.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np

from .model import DemandMatrix, ServerMatrix, ValidationError

# numpy view of ``fast_move`` (include/fastb200.h)
MOVE_DTYPE = np.dtype([("bytes", "<i8"), ("from_gpu", "<i4"), ("to_gpu", "<i4")])
# numpy view of ``fast_strip_rec``
STRIP_DTYPE = np.dtype([("real", "<i8"), ("stage", "<i4"), ("src", "<i2"), ("dst", "<i2")])


def stage_bytes_from_strip(weight: np.ndarray, perm: np.ndarray, strip: np.ndarray) -> np.ndarray:
    """Per-edge real bytes [k_raw, n] of the raw stages from the aux run-out
    table (fast_strip_rec): strip_auxiliary (birkhoff.py:225-252) charges a
    cell's aux before its real bytes, so every stage using an aux cell before
    the record's stage carries 0 real bytes, that stage carries `real`, and
    every other edge carries the full stage weight."""
    weight = np.asarray(weight, dtype=np.int64)
    sb = np.repeat(weight[:, None], perm.shape[1], axis=1)
    for rec in strip[strip["stage"] >= 0]:
        u, v, kl = int(rec["src"]), int(rec["dst"]), int(rec["stage"])
        ks = np.flatnonzero(perm[:kl, u] == v)
        sb[ks, u] = 0
        sb[kl, u] = int(rec["real"])
    return sb


def balanced_from_compact(D: np.ndarray, mask: np.ndarray, vals: np.ndarray, n: int,
                          m: int) -> np.ndarray:
    """Rebuild the balanced matrix from D and the compact cross-tile deltas
    (fast_compact_batch): bit p*m+q of mask[t] marks a changed cell of cross
    tile t (i-major order, j != i), vals holds their values in tile order
    then bit order."""
    bal = np.array(D, dtype=np.int64, copy=True)
    T = n * (n - 1)
    if T == 0:
        return bal
    bits = np.unpackbits(np.ascontiguousarray(mask).view(np.uint8).reshape(T, 8), axis=1,
                         bitorder="little")[:, : m * m]
    t_idx, bit = np.nonzero(bits)
    if len(vals) != len(t_idx):
        raise ValueError(f"compact result has {len(vals)} values for {len(t_idx)} changed cells")
    i = t_idx // (n - 1)
    jj = t_idx - i * (n - 1)
    j = jj + (jj >= i)
    p, q = bit // m, bit - (bit // m) * m
    bal[i * m + p, j * m + q] = vals
    return bal


@dataclass(frozen=True)
class IntraMove:
    """``bytes`` from ``from_gpu`` to ``to_gpu`` inside ``server`` (:37-56)."""

    server: int
    from_gpu: int
    to_gpu: int
    for_dst_server: int
    bytes: int

    def __post_init__(self) -> None:
        if self.from_gpu == self.to_gpu:
            raise ValidationError("intra move must change GPUs")
        if self.bytes <= 0:
            raise ValidationError("intra move must carry positive bytes")


@dataclass(frozen=True, eq=False)
class BalancePlan:
    """Phase-1 result: moves, scalar-tile matrix, redistribution tables."""

    moves: tuple[IntraMove, ...]
    reshaped: DemandMatrix
    redistribution: dict[tuple[int, int], np.ndarray]


@dataclass(frozen=True)
class PermutationStage:
    """One stage: partial matching of servers, edges sorted by (src, dst)."""

    weight: int
    edges: tuple[tuple[int, int, int], ...]

    def __post_init__(self) -> None:
        if self.weight < 0:
            raise ValidationError("stage weight must be non-negative")
        edges = tuple(sorted(self.edges, key=lambda e: (e[0], e[1])))
        object.__setattr__(self, "edges", edges)
        srcs = {e[0] for e in edges}
        dsts = {e[1] for e in edges}
        if len(srcs) != len(edges) or len(dsts) != len(edges):
            raise ValidationError("stage edges must form a partial matching")
        for _, _, b in edges:
            if b < 0 or b > self.weight:
                raise ValidationError("edge bytes must lie in [0, stage weight]")

    @property
    def matching(self) -> dict[int, int]:
        return {s: d for s, d, _ in self.edges}

    def max_edge_bytes(self) -> int:
        return max((b for _, _, b in self.edges), default=0)


@dataclass(frozen=True, eq=False)
class Decomposition:
    stages: tuple[PermutationStage, ...]
    aux: np.ndarray
    common_sum: int


@dataclass(frozen=True, eq=False)
class Schedule:
    plan: BalancePlan
    decomposition: Decomposition
    stages: tuple[PermutationStage, ...]


def _fast_stage(weight: int, edges: tuple) -> PermutationStage:
    """Build a stage whose edges are already sorted and valid (device output)."""
    st = object.__new__(PermutationStage)
    object.__setattr__(st, "weight", weight)
    object.__setattr__(st, "edges", edges)
    return st


@dataclass(frozen=True, eq=False)
class PackedSchedule:
    """Host copy of one matrix of the packed device layout."""

    n: int
    m: int
    status: int
    balanced: np.ndarray | None      # [G,G]
    server: np.ndarray | None        # [n,n]
    move_count: np.ndarray | None    # [T]
    moves: np.ndarray | None         # [T,S] structured MOVE_DTYPE
    common_sum: int
    aux: np.ndarray                  # [n,n]
    n_raw: int
    stage_weight: np.ndarray         # [n_raw]
    stage_perm: np.ndarray           # [n_raw,n] uint8
    stage_bytes: np.ndarray          # [n_raw,n]
    n_stages: int
    stage_order: np.ndarray          # [n_stages]

    # -- phase 1 --------------------------------------------------------
    def move_list(self) -> list[tuple[int, int, int, int, int]]:
        """(server, from, to, dst_server, bytes) in emission order."""
        out = []
        n = self.n
        t = 0
        mb, mf, mt = self.moves["bytes"], self.moves["from_gpu"], self.moves["to_gpu"]
        for i in range(n):
            for j in range(n):
                if i == j:
                    continue
                for s in range(int(self.move_count[t])):
                    out.append((i, int(mf[t, s]), int(mt[t, s]), j, int(mb[t, s])))
                t += 1
        return out

    def reshaped(self) -> np.ndarray:
        """Cross tiles collapsed to diag(row sums), intra tiles as-is."""
        n, m = self.n, self.m
        r = self.balanced.copy()
        for i in range(n):
            for j in range(n):
                if i == j:
                    continue
                blk = r[i * m:(i + 1) * m, j * m:(j + 1) * m]
                rows = blk.sum(axis=1)
                blk[...] = 0
                blk[np.arange(m), np.arange(m)] = rows
        return r

    def redistribution(self) -> dict[tuple[int, int], np.ndarray]:
        n, m = self.n, self.m
        out = {}
        for i in range(n):
            for j in range(n):
                if i != j:
                    out[(i, j)] = self.balanced[i * m:(i + 1) * m, j * m:(j + 1) * m].copy()
        return out

    def balance_plan(self) -> BalancePlan:
        moves = tuple(IntraMove(s, f, t, d, b) for s, f, t, d, b in self.move_list())
        reshaped = DemandMatrix(self.n, self.m, self.reshaped())
        return BalancePlan(moves=moves, reshaped=reshaped, redistribution=self.redistribution())

    # -- phase 2 --------------------------------------------------------
    def raw_stages(self) -> tuple[PermutationStage, ...]:
        """Decomposition-order stages, every edge carrying the full weight."""
        n = self.n
        return tuple(
            _fast_stage(int(w), tuple((u, int(self.stage_perm[k, u]), int(w)) for u in range(n)))
            for k, w in enumerate(self.stage_weight))

    def sorted_stages(self) -> tuple[PermutationStage, ...]:
        out = []
        for k in self.stage_order:
            k = int(k)
            row = self.stage_bytes[k]
            perm = self.stage_perm[k]
            edges = tuple((u, int(perm[u]), int(row[u])) for u in np.flatnonzero(row > 0).tolist())
            out.append(_fast_stage(int(self.stage_weight[k]), edges))
        return tuple(out)

    def decomposition(self) -> Decomposition:
        return Decomposition(stages=self.raw_stages(), aux=self.aux.copy(),
                             common_sum=int(self.common_sum))

    def to_schedule(self) -> Schedule:
        return Schedule(plan=self.balance_plan(), decomposition=self.decomposition(),
                        stages=self.sorted_stages())


# -- canonical JSON (pipeline.py:72-208) ----------------------------------

def dumps_canonical(payload: dict) -> str:
    return json.dumps(payload, sort_keys=True, separators=(",", ":"))


def _stages_json(stages) -> list[dict]:
    return [{"weight": int(st.weight), "edges": [[int(s), int(d), int(b)] for s, d, b in st.edges]}
            for st in stages]


def schedule_to_json(schedule: Schedule) -> str:
    """Byte-identical to tiersched.schedule_to_json for fast schedules."""
    plan = schedule.plan
    payload = {
        "scheduler": "fast",
        "n": plan.reshaped.n_servers,
        "m": plan.reshaped.gpus_per_server,
        "balance": {
            "moves": [{"server": mv.server, "from": mv.from_gpu, "to": mv.to_gpu,
                       "dst_server": mv.for_dst_server, "bytes": mv.bytes}
                      for mv in plan.moves],
            "reshaped": plan.reshaped.sizes.tolist(),
            "redist": {f"{i}->{j}": t.tolist() for (i, j), t in plan.redistribution.items()},
        },
        "common_sum": int(schedule.decomposition.common_sum),
        "aux": schedule.decomposition.aux.tolist(),
        "stages": _stages_json(schedule.stages),
    }
    return dumps_canonical(payload)


def schedule_from_json(text: str) -> Schedule:
    try:
        payload = json.loads(text)
    except json.JSONDecodeError as exc:
        raise ValidationError(f"schedule is not valid JSON: {exc}") from exc
    if payload.get("scheduler") != "fast":
        raise ValidationError(f"unknown scheduler kind: {payload.get('scheduler')!r}")
    try:
        n, m = int(payload["n"]), int(payload["m"])
        bal = payload["balance"]
        moves = tuple(IntraMove(int(x["server"]), int(x["from"]), int(x["to"]),
                                int(x["dst_server"]), int(x["bytes"])) for x in bal["moves"])
        reshaped = DemandMatrix(n, m, np.array(bal["reshaped"], dtype=np.int64))
        redist = {}
        for key, table in bal["redist"].items():
            i, j = key.split("->")
            redist[(int(i), int(j))] = np.array(table, dtype=np.int64)
        plan = BalancePlan(moves=moves, reshaped=reshaped, redistribution=redist)
        dec = Decomposition(stages=(), aux=np.array(payload["aux"], dtype=np.int64),
                            common_sum=int(payload["common_sum"]))
        stages = tuple(PermutationStage(int(x["weight"]),
                                        tuple((int(s), int(d), int(b)) for s, d, b in x["edges"]))
                       for x in payload["stages"])
    except (KeyError, TypeError, IndexError) as exc:
        raise ValidationError(f"malformed schedule document: {exc}") from exc
    return Schedule(plan=plan, decomposition=dec, stages=stages)


def server_matrix_of(p: PackedSchedule) -> ServerMatrix:
    return ServerMatrix(totals=p.server.copy())
