"""Row-batch layout of the private-dataset query.

The reference engine packs at most N/2 rows into one ciphertext per column
(pdq/columns.py:15-60 rejects more).  For larger datasets the rows are split
into blocks of N/2 rows; block b is encrypted and evaluated on rank
b % world with the reference circuit unchanged (pdq/engine.py:209-244 per
block), and only the final aggregates cross GPUs:

* ``sum``: every rank adds its blocks' rotate_sum outputs (ckks_add), then one
  all-reduce of the stacked residues plus one mod-q fix-up kernel
  (ShardGroup.all_reduce_ciphertexts) gives every rank the global total --
  the same words as ckks_add over all blocks on one GPU (modular addition is
  order-independent);
* ``avg``: total and count are reduced in the same all-reduce; the two-party
  inverse of the global count runs once, on rank 0;
* ``index`` / ``ratio`` are per-row: each rank returns its own blocks'
  results (no collective).

Block encryption randomness is Rng(seed + b), so block b's ciphertexts are
the same words whichever rank owns it.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from ..coremath.modmath import ParameterError
from ..coremath.sampling import Rng
from ..schemes.ckks import ckks_add
from .columns import encode_column
from .engine import PdqEngine, QueryResult, encrypt_query_constants, two_party_multiply_inverse
from .shard import ShardGroup


@dataclass
class BlockResult:
    agg: str
    cts: dict            # aggregates (sum/avg) or {block: {name: ct}} (index/ratio)
    blocks: list         # blocks evaluated on this rank
    meta: dict


class RowBlockEngine:
    def __init__(self, ev, cfg, group: ShardGroup | None = None):
        self.ev, self.cfg = ev, cfg
        self.group = group or ShardGroup(0, 1)
        self.slots = ev.slots
        self.engines: dict[int, PdqEngine] = {}
        self.total_rows = 0
        self.nblocks = 0

    def blocks_of_rank(self) -> list[int]:
        return [b for b in range(self.nblocks) if self.group.owner(b) == self.group.rank]

    def load(self, data: dict, pk, seed: int = 1):
        """Encrypt the columns of this rank's row blocks (data: name -> rows)."""
        rows = len(next(iter(data.values())))
        self.total_rows = rows
        self.nblocks = (rows + self.slots - 1) // self.slots
        if self.nblocks < self.group.world:
            raise ParameterError(f"{self.nblocks} row blocks for {self.group.world} ranks")
        for b in self.blocks_of_rank():
            lo, hi = b * self.slots, min(rows, (b + 1) * self.slots)
            cfg_b = replace(self.cfg, rows=hi - lo)
            eng = PdqEngine(self.ev, cfg_b)
            rng = Rng(int(seed + b).to_bytes(32, "little"))
            for name, vals in data.items():
                eng.add_column(encode_column(self.ev, cfg_b, name, vals[lo:hi], pk, rng))
            self.engines[b] = eng

    def run(self, spec, pk, channel=None, const_seed: int = 7,
            rng: np.random.Generator | None = None) -> BlockResult:
        ev = self.ev
        temps = encrypt_query_constants(ev, self.cfg, spec, pk,
                                        Rng(int(const_seed).to_bytes(32, "little")))
        mine = self.blocks_of_rank()
        if spec.agg in ("index", "ratio"):
            out = {b: self.engines[b].run(spec, channel=channel, temps=temps, rng=rng).cts
                   for b in mine}
            return BlockResult(spec.agg, out, mine, {})
        if spec.agg not in ("sum", "avg"):
            raise ParameterError(f"unknown aggregator {spec.agg!r}")
        totals, counts = [], []
        for b in mine:
            eng = self.engines[b]
            mask = eng.predicate_mask(spec.predicate, temps)
            totals.append(ev.rotate_sum(ev.mul(mask, eng._column(spec.col, temps).value)))
            if spec.agg == "avg":
                counts.append(ev.rotate_sum(mask, pre_vec=eng.validity))
        aggs = [_sum_all(ev, totals)] + ([_sum_all(ev, counts)] if counts else [])
        aggs = self.group.all_reduce_ciphertexts(ev.ctx, aggs)
        if spec.agg == "sum":
            return BlockResult("sum", {"sum": aggs[0]}, mine, {})
        total, count = aggs
        cts = {"count": count, "total": total}
        meta = {}
        if self.group.rank == 0 and channel is not None:
            inv, flags = two_party_multiply_inverse(ev, self.cfg, count, channel, rng)
            cts["avg"] = ev.mul(total, inv)
            meta["recip_flags"] = flags.tolist()
        return BlockResult("avg", cts, mine, meta)


def _sum_all(ev, cts):
    acc = cts[0]
    for c in cts[1:]:
        acc = ckks_add(ev.ctx, acc, c)
    return acc


def as_query_result(res: BlockResult) -> QueryResult:
    return QueryResult(res.agg, res.cts, res.meta)
