"""Multi-GPU sharding of the pair space.

Pairs are independent, so the path shards with no data-path collective: each
rank featurizes and predicts its own slice, and the only exchange is one
all-gather of the fp32 predictions at the end (`torch.distributed`
all_gather_into_tensor = ncclAllGather over NVLink with the NCCL backend; gloo
on CPU for the tests).

Global pair order is spec-major, p = g * C + c (the SP_PAIRS_CROSS order).
  axis="config": rank r takes configs [C*r/W, C*(r+1)/W) x all specs; its local
                 layout is [g][c_local] (what sp_featurize CROSS writes for the
                 config slice), padded to ceil(C/W) configs.
  axis="spec":   rank r takes specs [G*r/W, G*(r+1)/W) x all configs; local
                 layout [g_local][c], padded to ceil(G/W) specs.  Concatenating
                 ranks in order is the global order (plus padding).
All-gather needs equal counts, hence the padding; padded slots are NaN and
are dropped when the global array is assembled.
"""
from __future__ import annotations

from dataclasses import dataclass

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

    def __post_init__(self):
        assert self.axis in ("config", "spec")
        assert 0 <= self.rank < self.world

    # ---- this rank's slice
    @property
    def config_range(self) -> tuple[int, int]:
        if self.axis == "config":
            return shard_bounds(self.n_configs, self.rank, self.world)
        return 0, self.n_configs

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
    def padded_pairs(self) -> int:
        """Per-rank buffer length (equal on every rank)."""
        if self.axis == "config":
            return -(-self.n_configs // self.world) * self.n_specs
        return -(-self.n_specs // self.world) * self.n_configs

    # ---- local <-> global index maps
    def rank_global_index(self, rank: int) -> np.ndarray:
        """Global pair index of every padded local slot of `rank` (-1 = padding)."""
        s = Sharder(self.n_configs, self.n_specs, self.world, rank, self.axis)
        c0, c1 = s.config_range
        g0, g1 = s.spec_range
        out = np.full(self.padded_pairs, -1, dtype=np.int64)
        if self.axis == "config":
            n_pad = self.padded_pairs // self.n_specs
            for g in range(self.n_specs):
                loc = g * (c1 - c0) + np.arange(c1 - c0)
                out[loc] = g * self.n_configs + np.arange(c0, c1)
            del n_pad
        else:
            loc = np.arange((g1 - g0) * self.n_configs)
            out[loc] = g0 * self.n_configs + loc
        return out

    def global_index(self) -> np.ndarray:
        """[world * padded_pairs] global index of the all-gathered buffer (-1 = padding)."""
        return np.concatenate([self.rank_global_index(r) for r in range(self.world)])


def pad_local(local: torch.Tensor, sharder: Sharder) -> torch.Tensor:
    out = torch.full((sharder.padded_pairs,), float("nan"), dtype=local.dtype, device=local.device)
    out[: local.numel()] = local
    return out


def all_gather_predictions(local: torch.Tensor, sharder: Sharder, group=None,
                           gathered: torch.Tensor | None = None) -> torch.Tensor:
    """One all-gather of every rank's padded predictions, reassembled into the
    global spec-major order (length n_specs * n_configs) on every rank."""
    import torch.distributed as dist

    buf = local if local.numel() == sharder.padded_pairs else pad_local(local, sharder)
    if gathered is None:
        gathered = torch.empty(sharder.world * sharder.padded_pairs, dtype=buf.dtype, device=buf.device)
    dist.all_gather_into_tensor(gathered, buf, group=group)
    idx = torch.from_numpy(sharder.global_index()).to(buf.device)
    keep = idx >= 0
    out = torch.empty(sharder.n_specs * sharder.n_configs, dtype=buf.dtype, device=buf.device)
    out[idx[keep]] = gathered[keep]
    return out


def predict_sharded(ctx, batch, spec_array, model, sharder: Sharder, group=None, stream=None,
                    gather: bool = True):
    """This rank's slice through sp_featurize + sp_predict on its GPU, then the
    all-gather.  `batch` is the full host ConfigBatch (every rank holds the
    same inputs; only the slice is uploaded)."""
    from . import api

    c0, c1 = sharder.config_range
    g0, g1 = sharder.spec_range
    local_batch = batch.subset(np.arange(c0, c1)) if (c0, c1) != (0, batch.n_configs) else batch
    specs = ctx.load_gpu_specs(spec_array)
    db = api.DeviceBatch.from_host(local_batch, ctx.torch_device)
    n = (g1 - g0) * local_batch.n_configs
    feats = api.Features.empty(local_batch.family, n, ctx.torch_device)
    lat = torch.empty(sharder.padded_pairs, dtype=torch.float32, device=ctx.torch_device)
    lat.fill_(float("nan"))
    ctx.featurize(db, specs, feats, api.cross(g0, g1), stream)
    ctx.predict(model, feats, lat, None, stream)
    if not gather:
        return lat[:n]
    return all_gather_predictions(lat, sharder, group)
