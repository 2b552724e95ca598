"""World-size-2 gloo test of the data-parallel path on CPU: each rank takes its contiguous shard,
computes the covariance partials, packs them in the C-ABI's packed layout (blk_off from a host-only plan),
all-reduces them, and finalises.  The result must equal the single-process covariance of the whole set.
Also checks that the seeded generator is shard-invariant (image i does not depend on the shard)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_1412_0781_b200 as F
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _pack(plan, S, s0, n):
    buf = np.zeros(plan.n_partial)
    for k, Sk in enumerate(S):
        buf[plan.blk_off[k]:plan.blk_off[k + 1]] = Sk[np.triu_indices(Sk.shape[0])]
    buf[plan.n_blk:plan.n_blk + len(s0)] = s0
    buf[-1] = n
    return buf


def _unpack_and_finalize(plan, buf):
    S = F.unpack_blocks(plan, buf[:plan.n_blk])
    s0 = buf[plan.n_blk:plan.n_blk + int(plan.p[0])]
    return O.finalize_covariance(S, s0, int(round(buf[-1])))


def _worker(rank, world, port, n, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.config("C2")
    plan = F.fbspca_plan(cfg["L"], cfg["c"], cfg["R"], device=-1)
    basis = O.build_basis(cfg["c"], cfg["R"])
    s, e = F.shard_range(n, rank, world)
    sigma = synth.blobs.noise_sigma(cfg)
    imgs = synth.blob_images(cfg, s, e - s, sigma_n=sigma).double().numpy()
    A = O.expand(imgs, basis)
    S, s0, cnt = O.covariance_partials(A)
    buf = torch.from_numpy(_pack(plan, S, s0, cnt))
    dist.all_reduce(buf)
    mean, C = _unpack_and_finalize(plan, buf.numpy())
    if rank == 0:
        out.put((mean, C))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_covariance_equals_single_process():
    n = 24
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    mean_d, C_d = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = synth.config("C2")
    basis = O.build_basis(cfg["c"], cfg["R"])
    imgs = synth.blob_images(cfg, 0, n).double().numpy()
    mean, C = O.block_covariance(O.expand(imgs, basis))
    assert np.allclose(mean, mean_d, rtol=0, atol=1e-12 * np.abs(mean).max())
    for a, b in zip(C, C_d):
        assert np.max(np.abs(a - b)) <= 1e-11 * max(1.0, np.abs(a).max())


def test_generator_is_shard_invariant():
    cfg = synth.config("C3")
    sig = 1.0
    full = synth.blob_images(cfg, 0, 40, sigma_n=sig)
    parts = torch.cat([synth.blob_images(cfg, s, e - s, sigma_n=sig) for s, e in ((0, 13), (13, 31), (31, 40))])
    assert torch.equal(full, parts)
    a = synth.c1_images(6, first=0)
    b = np.concatenate([synth.c1_images(2, first=0), synth.c1_images(4, first=2)])
    assert np.array_equal(a, b)
