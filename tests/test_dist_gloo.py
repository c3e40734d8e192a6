"""Multi-rank path on CPU: world_size 2 over gloo (SURVEY §8(e) verification:
the gathered result must equal the single-process result byte for byte).
The per-rank compute is the fp64 oracle here (no GPU in the CPU suite); the
sharding, padding, all-gather and reassembly are the product code of
paper_2601_14910_b200/dist.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


from paper_2601_14910_b200 import dist as D  # noqa: E402  (loads libsynperf.so; no GPU call)


@pytest.mark.parametrize("axis", ["config", "spec"])
@pytest.mark.parametrize("n_configs,n_specs,world", [(10, 3, 2), (7, 11, 4), (1, 5, 3), (33, 1, 8)])
def test_index_maps_partition_the_pairs(axis, n_configs, n_specs, world):
    s = D.Sharder(n_configs, n_specs, world, 0, axis)
    idx = s.global_index()
    real = idx[idx >= 0]
    assert np.array_equal(np.sort(real), np.arange(n_configs * n_specs))
    total = 0
    for r in range(world):
        sr = D.Sharder(n_configs, n_specs, world, r, axis)
        assert sr.padded_pairs == s.padded_pairs
        assert sr.local_pairs <= sr.padded_pairs
        total += sr.local_pairs
    assert total == n_configs * n_specs


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, axis, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from workloads import gen, models, specs

        b = gen.gen_attention(9, 8, 5, max_bs=3, qlen_max=1500, kvlen_max=2500)
        sa = specs.paper_gpu_specs()
        model = models.random_mlp(b.family, 7)
        sh = D.Sharder(b.n_configs, len(sa), world, rank, axis)
        c0, c1 = sh.config_range
        g0, g1 = sh.spec_range
        cl, gl = O.cross_pairs(c1 - c0, (g0, g1))
        f = O.featurize(b, sa, cfg_idx=cl + c0, spec_idx=gl)
        lat, _, _ = O.predict(model, f)
        local = torch.from_numpy(lat.astype(np.float32))
        full = D.all_gather_predictions(local, sh)
        if rank == 0:
            np.save(out_path, full.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("axis", ["config", "spec"])
def test_gloo_world2_allgather_matches_single_process(tmp_path, orc, axis):
    from workloads import gen, models, specs

    out = str(tmp_path / "gathered.npy")
    mp.start_processes(_worker, args=(2, _free_port(), axis, out), nprocs=2, join=True, start_method="spawn")
    got = np.load(out)
    b = gen.gen_attention(9, 8, 5, max_bs=3, qlen_max=1500, kvlen_max=2500)
    sa = specs.paper_gpu_specs()
    lat, _, _ = orc.predict(models.random_mlp(b.family, 7), orc.featurize(b, sa))
    assert np.array_equal(got, lat.astype(np.float32), equal_nan=True)
