"""Multi-rank path on CPU: world_size 2-3 over gloo (SURVEY §8(e) verification:
the gathered result must equal the single-process result byte for byte).
The per-rank compute is the fp64 oracle here (no GPU in the CPU suite); the
sharding (seeded config shuffle, spec ranges), padding, chunked all-gather and
reassembly are the product code of paper_2601_14910_b200/dist.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


from paper_2601_14910_b200 import dist as D  # noqa: E402  (loads libsynperf.so; no GPU call)


@pytest.mark.parametrize("axis", ["config", "spec"])
@pytest.mark.parametrize("seed", [None, 3])
@pytest.mark.parametrize("chunks", [1, 3])
@pytest.mark.parametrize("n_configs,n_specs,world", [(10, 3, 2), (7, 11, 4), (1, 5, 3), (33, 1, 8), (5, 4, 8)])
def test_index_maps_partition_the_pairs(axis, seed, chunks, n_configs, n_specs, world):
    s = D.Sharder(n_configs, n_specs, world, 0, axis, seed, chunks)
    idx = s.global_index()
    assert idx.shape == (world * s.padded_pairs,)
    real = idx[idx >= 0]
    assert np.array_equal(np.sort(real), np.arange(n_configs * n_specs))
    total = 0
    seen = []
    for r in range(world):
        sr = D.Sharder(n_configs, n_specs, world, r, axis, seed, chunks)
        assert sr.padded_pairs == s.padded_pairs and sr.block == s.block
        assert sr.local_pairs <= sr.padded_pairs
        assert sr.chunk_bounds() == s.chunk_bounds() and sr.chunk_offsets()[-1] == sr.padded_pairs
        total += sr.local_pairs
        seen.append(sr.configs)
    assert total == n_configs * n_specs
    if axis == "config":  # the ranks' configs partition the (shuffled) config axis
        assert np.array_equal(np.sort(np.concatenate(seen)), np.arange(n_configs))


def test_seeded_shuffle_is_rank_independent():
    a = D.Sharder(1000, 11, 4, 0, "config", seed=7)
    b = D.Sharder(1000, 11, 4, 3, "config", seed=7)
    assert np.array_equal(a.perm, b.perm) and not np.array_equal(a.perm, np.arange(1000))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, axis, seed, chunks, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from workloads import gen, models, specs

        b = gen.gen_attention(9, 8, 5, max_bs=3, qlen_max=1500, kvlen_max=2500)
        sa = specs.paper_gpu_specs()
        model = models.random_mlp(b.family, 7)
        sh = D.Sharder(b.n_configs, len(sa), world, rank, axis, seed, chunks)
        cfg = sh.configs if axis == "config" else np.arange(b.n_configs)
        g0, g1 = sh.spec_range
        local = torch.full((sh.padded_pairs,), float("nan"), dtype=torch.float32)

        def compute(k):  # this rank's real part of chunk k: spec rows x local configs
            a0, a1, b0, b1 = sh.chunk_bounds()[k]
            nr, ncol = sh.real_extent(k)
            if nr == 0 or ncol == 0:
                return
            gl = np.repeat(np.arange(g0 + a0, g0 + a0 + nr, dtype=np.int32), ncol)
            cl = np.tile(cfg[b0:b0 + ncol], nr)
            f = O.featurize(b, sa, cfg_idx=cl, spec_idx=gl)
            lat, _, _ = O.predict(model, f)
            D.place_local(torch.from_numpy(lat.astype(np.float32)), sh, local, k)

        gathered = torch.empty(world * sh.padded_pairs, dtype=torch.float32)
        D.all_gather_chunks(local, sh, gathered, compute=compute)
        full = D.assemble(gathered, sh)
        if rank == 0:
            np.save(out_path, full.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("axis,seed,chunks,world", [("config", None, 1, 2), ("config", 11, 3, 2),
                                                     ("spec", None, 2, 2), ("config", 5, 4, 3)])
def test_gloo_chunked_allgather_matches_single_process(tmp_path, orc, axis, seed, chunks, world):
    from workloads import gen, models, specs

    out = str(tmp_path / "gathered.npy")
    mp.start_processes(_worker, args=(world, _free_port(), axis, seed, chunks, out), nprocs=world, join=True,
                       start_method="spawn")
    got = np.load(out)
    b = gen.gen_attention(9, 8, 5, max_bs=3, qlen_max=1500, kvlen_max=2500)
    sa = specs.paper_gpu_specs()
    lat, _, _ = orc.predict(models.random_mlp(b.family, 7), orc.featurize(b, sa))
    assert np.array_equal(got, lat.astype(np.float32), equal_nan=True)


def test_all_gather_predictions_unpadded_local(tmp_path, orc):
    """all_gather_predictions accepts a dense (unpadded) local result."""
    out = str(tmp_path / "g.npy")
    mp.start_processes(_worker_dense, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    from workloads import gen, models, specs

    b = gen.gen_gemm(13, 8)
    sa = specs.paper_gpu_specs()
    lat, _, _ = orc.predict(models.random_mlp(b.family, 2), orc.featurize(b, sa))
    assert np.array_equal(np.load(out), lat.astype(np.float32), equal_nan=True)


def _worker_dense(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from workloads import gen, models, specs

        b = gen.gen_gemm(13, 8)
        sa = specs.paper_gpu_specs()
        sh = D.Sharder(b.n_configs, len(sa), world, rank, "config", seed=1, chunks=2)
        cfg = sh.configs
        gl = np.repeat(np.arange(len(sa), dtype=np.int32), len(cfg))
        cl = np.tile(cfg, len(sa))
        lat, _, _ = O.predict(models.random_mlp(b.family, 2), O.featurize(b, sa, cfg_idx=cl, spec_idx=gl))
        full = D.all_gather_predictions(torch.from_numpy(lat.astype(np.float32)), sh)
        if rank == 0:
            np.save(out_path, full.numpy())
    finally:
        dist.destroy_process_group()
