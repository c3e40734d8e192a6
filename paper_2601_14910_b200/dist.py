"""Multi-GPU sharding of the pair space.

Pairs are independent, so the path shards with no data-path collective: each
rank featurizes and predicts its own slice, and the only exchange is the
all-gather of the fp32 predictions (`torch.distributed`
all_gather_into_tensor = ncclAllGather over NVLink with the NCCL backend; gloo
on CPU for the tests).

Global pair order is spec-major, p = g * C + c (the SP_PAIRS_CROSS order).
  axis="config": a seeded permutation `perm` of the configs (cost balance:
                 attention configs range over five orders of magnitude of
                 tasks), then rank r takes permuted configs
                 perm[C*r/W : C*(r+1)/W] x all specs.  Its local block is
                 [A = G][B = ceil(C/W)] (spec-major, padded configs).
  axis="spec":   rank r takes specs [G*r/W, G*(r+1)/W) x all configs (spec-major
                 order makes it a contiguous slice of the global output); local
                 block [A = ceil(G/W)][B = C].
The exchange overlaps the compute: the local block is cut into K chunks --
along the configs for the config axis (an attention launch walks each
config's tasks once for all its specs, so cutting the specs would repeat that
walk per chunk), along the specs for the spec axis -- with the same bounds on
every rank, so the all-gather counts match.  The local buffer is chunk-major
(chunk k's [rows][cols] block after chunk k-1's); chunk k's predictions are
all-gathered on a communication stream while chunk k+1 is computed.  Padded
slots are NaN.  `global_index()` maps every slot of the gathered buffer --
chunk-major [k][rank][rows][cols] -- to its global pair (-1 = padding), so the
gathered buffer plus that map is the full result; assemble() scatters it into
the global order.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    return n * rank // world, n * (rank + 1) // world


@dataclass
class Sharder:
    n_configs: int
    n_specs: int
    world: int
    rank: int
    axis: str = "config"
    seed: int | None = None  # config axis: seeded shuffle of the configs (None: identity)
    chunks: int = 1          # all-gather chunks along the local spec dimension
    perm: np.ndarray = field(init=False, repr=False)

    def __post_init__(self):
        assert self.axis in ("config", "spec")
        assert 0 <= self.rank < self.world and self.chunks >= 1
        if self.axis == "config" and self.seed is not None:
            self.perm = np.random.default_rng(self.seed).permutation(self.n_configs).astype(np.int64)
        else:
            self.perm = np.arange(self.n_configs, dtype=np.int64)

    def _for(self, rank: int) -> "Sharder":
        s = Sharder.__new__(Sharder)
        s.__dict__.update(self.__dict__)
        s.rank = rank
        return s

    # ---- this rank's slice
    @property
    def config_range(self) -> tuple[int, int]:
        """Range of positions in `perm` (config axis) or of configs (spec axis)."""
        if self.axis == "config":
            return shard_bounds(self.n_configs, self.rank, self.world)
        return 0, self.n_configs

    @property
    def configs(self) -> np.ndarray:
        """Global config indices of this rank, in local order."""
        c0, c1 = self.config_range
        return self.perm[c0:c1]

    @property
    def spec_range(self) -> tuple[int, int]:
        if self.axis == "spec":
            return shard_bounds(self.n_specs, self.rank, self.world)
        return 0, self.n_specs

    @property
    def local_pairs(self) -> int:
        c0, c1 = self.config_range
        g0, g1 = self.spec_range
        return (c1 - c0) * (g1 - g0)

    @property
    def block(self) -> tuple[int, int]:
        """(A, B): the padded local block, [spec][config], equal on every rank."""
        if self.axis == "config":
            return self.n_specs, -(-self.n_configs // self.world)
        return -(-self.n_specs // self.world), self.n_configs

    @property
    def padded_pairs(self) -> int:
        """Per-rank buffer length (equal on every rank)."""
        a, b = self.block
        return a * b

    def chunk_bounds(self) -> list[tuple[int, int, int, int]]:
        """(a0, a1, b0, b1) of each all-gather chunk in the padded [A][B] block
        (the same on every rank): config ranges for the config axis, spec ranges
        for the spec axis."""
        A, B = self.block
        if self.axis == "config":
            k = max(1, min(self.chunks, B))
            return [(0, A, B * i // k, B * (i + 1) // k) for i in range(k)]
        k = max(1, min(self.chunks, A))
        return [(A * i // k, A * (i + 1) // k, 0, B) for i in range(k)]

    def chunk_offsets(self) -> list[int]:
        """Start of each chunk in the chunk-major local buffer (+ the total)."""
        off = [0]
        for a0, a1, b0, b1 in self.chunk_bounds():
            off.append(off[-1] + (a1 - a0) * (b1 - b0))
        return off

    # ---- local <-> global index maps
    def _local_global(self, rank: int) -> np.ndarray:
        """[A][B] global pair index of every padded slot of `rank` (-1 = padding)."""
        s = self._for(rank)
        A, B = self.block
        out = np.full((A, B), -1, dtype=np.int64)
        g0, g1 = s.spec_range
        cfg = s.configs if self.axis == "config" else np.arange(self.n_configs, dtype=np.int64)
        ng = g1 - g0
        out[:ng, :len(cfg)] = (np.arange(g0, g1, dtype=np.int64)[:, None] * self.n_configs + cfg[None, :])
        return out

    def global_index(self) -> np.ndarray:
        """Global pair of every slot of the gathered buffer, chunk-major
        [k][rank][a1 - a0][b1 - b0] (-1 = padding)."""
        per_rank = [self._local_global(r) for r in range(self.world)]
        parts = []
        for a0, a1, b0, b1 in self.chunk_bounds():
            for r in range(self.world):
                parts.append(per_rank[r][a0:a1, b0:b1].reshape(-1))
        return np.concatenate(parts)

    def real_extent(self, k: int) -> tuple[int, int]:
        """(rows, cols) of chunk k this rank really computes (the rest is padding)."""
        a0, a1, b0, b1 = self.chunk_bounds()[k]
        c0, c1 = self.config_range
        g0, g1 = self.spec_range
        return max(0, min(a1, g1 - g0) - a0), max(0, min(b1, c1 - c0) - b0)


def place_local(lat_dense: torch.Tensor, sharder: Sharder, out: torch.Tensor, k: int = 0) -> None:
    """Copy this rank's dense [rows][cols] predictions of chunk k (its real
    extent) into chunk k's padded block of the chunk-major local buffer `out`."""
    a0, a1, b0, b1 = sharder.chunk_bounds()[k]
    off = sharder.chunk_offsets()[k]
    nr, ncol = sharder.real_extent(k)
    blk = out[off:off + (a1 - a0) * (b1 - b0)].view(a1 - a0, b1 - b0)
    blk[:nr, :ncol].copy_(lat_dense[:nr * ncol].view(nr, ncol))


def assemble(gathered: torch.Tensor, sharder: Sharder, index: torch.Tensor | None = None) -> torch.Tensor:
    """Scatter the gathered buffer into the global spec-major order."""
    idx = index if index is not None else torch.from_numpy(sharder.global_index()).to(gathered.device)
    keep = idx >= 0
    out = torch.empty(sharder.n_specs * sharder.n_configs, dtype=gathered.dtype, device=gathered.device)
    out[idx[keep]] = gathered[keep]
    return out


def all_gather_chunks(local: torch.Tensor, sharder: Sharder, gathered: torch.Tensor, group=None,
                      compute=None, comm_stream=None) -> None:
    """All-gather the chunk-major local buffer chunk by chunk into `gathered`
    (chunk-major [k][rank][...]).  compute(k), if given, fills chunk k of the
    local buffer first; on CUDA the all-gather of chunk k runs on `comm_stream`
    (ordered after chunk k's compute by an event) while chunk k+1 is computed
    on the current stream."""
    import torch.distributed as dist

    W = sharder.world
    cuda = local.is_cuda and comm_stream is not None
    cur = torch.cuda.current_stream(local.device) if cuda else None
    off = sharder.chunk_offsets()
    for k in range(len(off) - 1):
        if compute is not None:
            compute(k)
        src = local[off[k]:off[k + 1]]
        dst = gathered[W * off[k]:W * off[k + 1]]
        if cuda:
            ev = torch.cuda.Event()
            ev.record(cur)
            comm_stream.wait_event(ev)
            with torch.cuda.stream(comm_stream):
                dist.all_gather_into_tensor(dst, src, group=group)
        else:
            dist.all_gather_into_tensor(dst, src, group=group)
    if cuda:
        cur.wait_stream(comm_stream)


def all_gather_predictions(local: torch.Tensor, sharder: Sharder, group=None,
                           gathered: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather of every rank's predictions, reassembled into the global
    spec-major order on every rank.  `local`: this rank's dense result,
    [spec in spec_range][config in sharder.configs] (what sp_featurize CROSS
    writes for the shard)."""
    buf = torch.full((sharder.padded_pairs,), float("nan"), dtype=local.dtype, device=local.device)
    g0, g1 = sharder.spec_range
    c0, c1 = sharder.config_range
    dense = local[: (g1 - g0) * (c1 - c0)].view(g1 - g0, c1 - c0)
    for k, (a0, a1, b0, b1) in enumerate(sharder.chunk_bounds()):
        nr, ncol = sharder.real_extent(k)
        place_local(dense[a0:a0 + nr, b0:b0 + ncol].reshape(-1), sharder, buf, k)
    if gathered is None:
        gathered = torch.empty(sharder.world * sharder.padded_pairs, dtype=buf.dtype, device=buf.device)
    all_gather_chunks(buf, sharder, gathered, group)
    return assemble(gathered, sharder)


class ShardedPredictor:
    """A rank's share of the design space on its GPU: the shard's configs are
    uploaded once, the spec table and scratch are prepared once (sp_prepare),
    and every run() computes the shard chunk by chunk through
    sp_featurize_predict (the fused pass for the uniform families) with the
    chunked all-gather of the predictions overlapped on a comm stream."""

    def __init__(self, ctx, batch, spec_array, model, sharder: Sharder, group=None, specs=None):
        from . import api

        self.ctx, self.model, self.sh, self.group = ctx, model, sharder, group
        dev = ctx.torch_device
        cfg = sharder.configs
        same = sharder.axis == "spec" or (len(cfg) == batch.n_configs and np.array_equal(cfg, np.arange(len(cfg))))
        local_batch = batch if same else batch.subset(cfg)
        self.family = local_batch.family
        self.nc = local_batch.n_configs
        self.specs = specs if specs is not None else ctx.load_gpu_specs(spec_array)
        self.db = api.DeviceBatch.from_host(local_batch, dev)
        self.g0, self.g1 = sharder.spec_range
        n_max = max(r * c for r, c in (sharder.real_extent(k) for k in range(len(sharder.chunk_bounds()))))
        self.feats = api.Features.empty(self.family, max(n_max, 1), dev)
        self.dense = torch.empty(max(n_max, 1), dtype=torch.float32, device=dev)
        self.local = torch.full((max(sharder.padded_pairs, 1),), float("nan"), dtype=torch.float32, device=dev)
        self.gathered = self.local if sharder.world == 1 else \
            torch.empty(sharder.world * sharder.padded_pairs, dtype=torch.float32, device=dev)
        self.comm = torch.cuda.Stream(dev) if dev.type == "cuda" else None
        self.last = self.dense[:0]
        self._offsets = sharder.chunk_offsets()
        ctx.prepare(self.family, self.nc, self.specs, (self.g0, self.g1))
        self._index = None

    def _compute(self, k):
        from . import api

        a0, a1, b0, b1 = self.sh.chunk_bounds()[k]
        nr, ncol = self.sh.real_extent(k)
        if nr == 0 or ncol == 0:
            return
        n = nr * ncol
        self.feats.n_pairs = n
        direct = nr == a1 - a0 and ncol == b1 - b0  # no padding: the dense rows are the chunk's block
        out = self.local[self._offsets[k]:self._offsets[k] + n] if direct else self.dense[:n]
        db = self.db if (b0, b0 + ncol) == (0, self.nc) else self.db.slice(b0, b0 + ncol)
        self.ctx.featurize_predict(db, self.specs, self.model, self.feats, out, None,
                                   api.cross(self.g0 + a0, self.g0 + a0 + nr))
        if not direct:
            place_local(out, self.sh, self.local, k)
        self.last = out  # the chunk's latencies, dense [spec][config] like self.feats

    def run(self, gather: bool = True) -> torch.Tensor:
        """One pass over the shard; returns the gathered buffer (chunk-major,
        see Sharder.global_index) or, without gather, the local chunk-major block."""
        import torch.distributed as dist

        if not gather or self.sh.world == 1 or not dist.is_initialized():
            for k in range(len(self._offsets) - 1):
                self._compute(k)
            return self.local  # (world 1: the gathered buffer is the local block)
        all_gather_chunks(self.local, self.sh, self.gathered, self.group, self._compute, self.comm)
        return self.gathered

    def global_result(self) -> torch.Tensor:
        """The last run's predictions in the global spec-major order."""
        if self._index is None:
            self._index = torch.from_numpy(self.sh.global_index()).to(self.gathered.device)
        return assemble(self.gathered, self.sh, self._index)


def predict_sharded(ctx, batch, spec_array, model, sharder: Sharder, group=None, specs=None,
                    gather: bool = True) -> torch.Tensor:
    """One-shot convenience: ShardedPredictor(...).run(), reassembled into the
    global order (gather) or this rank's padded local block (no gather)."""
    p = ShardedPredictor(ctx, batch, spec_array, model, sharder, group, specs)
    out = p.run(gather)
    return p.global_result() if gather else out
