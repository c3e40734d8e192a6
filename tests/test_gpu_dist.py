"""Multi-GPU path on the GPU: ShardedPredictor (seeded config
shuffle or spec ranges, chunked all-gather on a comm stream) must give the
single-GPU result byte for byte.  The NCCL test needs >= 2 GPUs and skips
otherwise (the driver's GPU boxes have one; the gloo tests cover the
multi-rank host logic on CPU)."""
import os
import socket

import numpy as np
import pytest
import torch

from workloads import gen, models, specs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_14910_b200 as sp

    return sp


def single_gpu(sp, b, sa, model_d):
    ctx = sp.Context(0)
    sh = ctx.load_gpu_specs(sa)
    m = ctx.load_model(model_d, "fp16")
    db = sp.DeviceBatch.from_host(b, "cuda:0")
    n = len(sa) * b.n_configs
    f = sp.Features.empty(b.family, n, "cuda:0")
    lat = torch.empty(n, dtype=torch.float32, device="cuda:0")
    ctx.featurize_predict(db, sh, m, f, lat)
    torch.cuda.synchronize()
    return lat.cpu().numpy()


@pytest.mark.parametrize("axis,seed,chunks,fam", [("config", 7, 3, "attention"), ("config", None, 1, "moe"),
                                                  ("spec", None, 4, "gemm")])
def test_sharded_world1_equals_device_path(sp, axis, seed, chunks, fam):
    from paper_2601_14910_b200 import dist as D

    b = {"attention": lambda: gen.gen_attention(300, 300, 41, max_bs=4, qlen_max=3000, kvlen_max=5000),
         "moe": lambda: gen.gen_moe(500, 42), "gemm": lambda: gen.gen_gemm(400, 43)}[fam]()
    sa = specs.paper_gpu_specs() if axis == "config" else specs.hypothetical_sweep_specs(70)
    md = models.random_mlp(b.family, 9)
    ref = single_gpu(sp, b, sa, md)
    ctx = sp.Context(0)
    s = D.Sharder(b.n_configs, len(sa), 1, 0, axis, seed, chunks)
    p = D.ShardedPredictor(ctx, b, sa, ctx.load_model(md, "fp16"), s)
    p.run()
    got = p.global_result().cpu().numpy()
    assert np.array_equal(got, ref, equal_nan=True)
    p.run()  # a second pass reuses the buffers
    assert np.array_equal(p.global_result().cpu().numpy(), ref, equal_nan=True)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _nccl_worker(rank, world, port, out):
    import torch.distributed as dist

    import paper_2601_14910_b200 as sp
    from paper_2601_14910_b200 import dist as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        b = gen.gen_attention(300, 300, 41, max_bs=4, qlen_max=3000, kvlen_max=5000)
        sa = specs.paper_gpu_specs()
        ctx = sp.Context(rank)
        s = D.Sharder(b.n_configs, len(sa), world, rank, "config", seed=5, chunks=3)
        p = D.ShardedPredictor(ctx, b, sa, ctx.load_model(models.random_mlp(b.family, 9), "fp16"), s)
        p.run()
        full = p.global_result().cpu().numpy()
        if rank == 0:
            np.save(out, full)
    finally:
        dist.destroy_process_group()


def test_nccl_world2_equals_single_gpu(sp, tmp_path):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    import torch.multiprocessing as mp

    out = str(tmp_path / "g.npy")
    mp.start_processes(_nccl_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    b = gen.gen_attention(300, 300, 41, max_bs=4, qlen_max=3000, kvlen_max=5000)
    ref = single_gpu(sp, b, specs.paper_gpu_specs(), models.random_mlp(b.family, 9))
    assert np.array_equal(np.load(out), ref, equal_nan=True)
