"""Sharding the private-dataset query across GPUs.

One process per GPU (torch.distributed; NCCL over NVLink/NVSwitch in
production, gloo in the CPU tests).  Two layouts:

* (atom, digit) units (``map_units`` / ``map_units_batched``): unit i of the
  predicate is computed by rank i % world (compare_digit_columns' per-digit
  loop, reference pdq/compare.py:147-154, is independent across digits and
  atoms).  The results are then exchanged in ONE all-gather of a stacked
  word block (plus one all-gather of the small per-unit descriptors), so
  every rank holds every unit's ciphertexts and the trees, boolean combine,
  aggregation and inverse run identically everywhere: the answer is
  bit-identical to one GPU (the circuit consumes no randomness).
* row blocks (``all_reduce_ciphertexts``, used by pdq/rowblocks.py): for
  datasets with more rows than slots every rank evaluates the whole circuit
  on its own row-block ciphertexts and the aggregates are summed with one
  all-reduce of the stacked residues (int64 SUM, exact for world <= 8 since
  every residue is < 2^60 / 8) followed by one mod-q fix-up launch
  (fhe_ewise EW_REDUCE): the same words as ckks_add over all blocks.

Received ciphertexts are views into the gathered block on this rank's own
device (torch.cuda.current_device()).
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass
class ShardGroup:
    rank: int
    world: int
    pg: object = None          # torch.distributed process group (None: default)

    @classmethod
    def from_env(cls):
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            return cls(dist.get_rank(), dist.get_world_size())
        return cls(0, 1)

    def owner(self, i: int) -> int:
        return i % self.world

    def map_units(self, units: list, fn):
        """Run fn(unit) for the units this rank owns, then exchange every
        result (a tuple of ciphertext-like objects or None) so all ranks hold
        all of them."""
        results = [fn(u) if self.owner(i) == self.rank else None for i, u in enumerate(units)]
        if self.world == 1:
            return results
        return self._exchange(results)

    def map_units_batched(self, units: list, fn, batch_fn, key, lanes=None):
        """map_units, but the units a rank owns are grouped by key(unit) and
        each group goes to batch_fn(list of units) (one lockstep batch);
        batch_fn may return None to fall back to fn per unit.  With a
        StreamPool (``lanes``, the context's worker pool) the independent
        groups run on separate CUDA streams and join on the caller's stream."""
        mine = [i for i in range(len(units)) if self.owner(i) == self.rank]
        groups: dict = {}
        for i in mine:
            groups.setdefault(key(units[i]), []).append(i)
        results: list = [None] * len(units)

        def run_group(idx):
            res = batch_fn([units[i] for i in idx]) if len(idx) > 1 else None
            if res is None:
                res = [fn(units[i]) for i in idx]
            for i, r in zip(idx, res):
                results[i] = r

        if lanes is not None and len(groups) > 1:
            lanes.run([lambda idx=idx: run_group(idx) for idx in groups.values()])
        else:
            for idx in groups.values():
                run_group(idx)
        if self.world == 1:
            return results
        return self._exchange(results)

    # -- exchange -------------------------------------------------------------
    def _backend_is_nccl(self) -> bool:
        import torch.distributed as dist

        return dist.get_backend(self.pg) == "nccl"

    def _exchange(self, results: list) -> list:
        """One all_gather_object of the descriptors + one all-gather of the
        stacked int64 words of every unit result."""
        import torch
        import torch.distributed as dist

        mine = [(i, res) for i, res in enumerate(results) if self.owner(i) == self.rank]
        descs = [(i, [_describe(ct) for ct in res]) for i, res in mine]
        all_descs: list = [None] * self.world
        dist.all_gather_object(all_descs, descs, group=self.pg)
        words = [sum(_words(d) for _, ds in rd for d in ds) for rd in all_descs]
        width = max(max(words), 1)
        kinds = {d[0] for rd in all_descs for _, ds in rd for d in ds if d is not None}
        device = (torch.device("cuda", torch.cuda.current_device())
                  if "ckks" in kinds or self._backend_is_nccl() else torch.device("cpu"))
        block = torch.zeros(width, dtype=torch.int64, device=device)
        off = 0
        for _, res in mine:
            for ct in res:
                if ct is None:
                    continue
                flat = _payload(ct)
                block[off:off + flat.numel()] = flat
                off += flat.numel()
        gathered = self._all_gather(block)
        out = list(results)
        for r, rd in enumerate(all_descs):
            if r == self.rank:
                continue
            off = 0
            for i, ds in rd:
                cts = []
                for d in ds:
                    if d is None:
                        cts.append(None)
                        continue
                    w = _words(d)
                    cts.append(_rebuild(d, gathered[r][off:off + w]))
                    off += w
                out[i] = tuple(cts)
        return out

    def _all_gather(self, block):
        """[world] tensors of block's shape; NCCL gathers on the device, gloo
        stages device blocks through host memory."""
        import torch
        import torch.distributed as dist

        if block.is_cuda and self._backend_is_nccl():
            flat = torch.empty(self.world * block.numel(), dtype=block.dtype, device=block.device)
            dist.all_gather_into_tensor(flat, block, group=self.pg)
            return list(flat.view(self.world, -1))
        host = block.cpu()
        parts = [torch.empty_like(host) for _ in range(self.world)]
        dist.all_gather(parts, host, group=self.pg)
        return [p.to(block.device) for p in parts]

    def all_reduce_ciphertexts(self, ctx, cts: list):
        """Sum same-shaped ciphertexts across ranks, slot-wise exact: one
        all-reduce (SUM) of their stacked residues, then one mod-q fix-up
        launch.  Returns new ciphertexts (inputs untouched); world 1 returns
        the inputs."""
        import torch
        import torch.distributed as dist

        if self.world == 1:
            return list(cts)
        if self.world > 8:
            raise ValueError("row-block aggregate is exact for at most 8 ranks")
        from ..rnspoly import CData
        from ..schemes.ckks import CkksCiphertext

        parts = [ct.data.view().reshape(-1) for ct in cts]
        stacked = torch.cat(parts)
        if stacked.is_cuda and self._backend_is_nccl():
            dist.all_reduce(stacked, op=dist.ReduceOp.SUM, group=self.pg)
        else:
            host = stacked.cpu()
            dist.all_reduce(host, op=dist.ReduceOp.SUM, group=self.pg)
            stacked.copy_(host)
        out, off = [], 0
        for ct in cts:
            d = ct.data
            flat = stacked[off:off + d.size]
            off += d.size
            cd = CData.wrap(flat, d.size_poly, d.size_modulus, d.n, d.domains[0])
            _reduce_rows(ctx, cd)
            out.append(CkksCiphertext(cd, ct.scale, ct.level))
        return out


def _reduce_rows(ctx, cd):
    """x mod q_j in place for every row of cd (the summed residues, < 8 q)."""
    from .. import _native
    from ..rnspoly import ew

    ew(ctx.chain, _native.EW_REDUCE, cd.view(), cd.view(), rows=cd.size_poly * cd.size_modulus,
       limbs=cd.size_modulus)


def _describe(ct):
    """Metadata needed to rebuild each ciphertext on the receivers (no device:
    every rank rebuilds on its own)."""
    if ct is None:
        return None
    if hasattr(ct, "data") and hasattr(ct.data, "size_poly"):
        d = ct.data
        return ("ckks", d.size_poly, d.size_modulus, d.n, d.domains[0].value, ct.scale, ct.level)
    if str(ct.dtype) != "torch.int64":
        raise TypeError("exchanged tensors must be int64")
    return ("tensor", tuple(ct.shape))


def _words(d) -> int:
    if d is None:
        return 0
    if d[0] == "ckks":
        return d[1] * d[2] * d[3]
    n = 1
    for s in d[1]:
        n *= s
    return n


def _rebuild(d, flat):
    if d[0] == "tensor":
        return flat.reshape(d[1]).clone()
    from ..rnspoly import CData, Domain
    from ..schemes.ckks import CkksCiphertext

    _, polys, limbs, n, domain, scale, level = d
    return CkksCiphertext(CData.wrap(flat, polys, limbs, n, Domain(domain)), scale, level)


def _payload(ct):
    # the ciphertext's words only (a resized CData keeps a larger buffer)
    return ct.data.view().reshape(-1) if hasattr(ct, "scale") else ct.reshape(-1)
