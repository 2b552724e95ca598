"""The collective half of K5 on hardware ("each worker is allocated a subset of the
images"): a 1-rank NCCL communicator through the library's own plumbing, the NCCL-registered partial buffer,
asynchronous-error polling, and the CUDA-graph form of the step.  (Multi-rank reduction arithmetic is covered
on the CPU by tests/test_distributed_cpu.py; the pool gives one GPU per call.)"""
import numpy as np
import pytest
import torch

import paper_1412_0781_b200 as F
import synth

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0") if torch.cuda.is_available() else None


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as g
    g.build()


@pytest.fixture(scope="module")
def c2():
    cfg = synth.config("C2")
    n = 3000
    imgs = synth.blob_images(cfg, 0, n, device=DEV)
    plan = F.fbspca_plan(cfg["L"], cfg["c"], cfg["R"], device=0, max_batch=1024)
    coeffs = F.fbspca_expand(plan, imgs)
    torch.cuda.synchronize()
    return plan, imgs, coeffs


def test_one_rank_nccl_covariance_equals_local(c2):
    """fbspca_nccl_unique_id -> fbspca_comm_init(1 rank) -> fbspca_covariance(comm): K5 writes into the
    registered buffer, the in-place ncclAllReduce runs, finalise reads it -- bit-identical to comm = NULL
    (a 1-rank sum is exact)."""
    plan, _, coeffs = c2
    b0, m0 = F.fbspca_covariance(plan, coeffs)
    comm = F.fbspca_comm_init(F.fbspca_nccl_unique_id(), 1, 0)
    try:
        stream = torch.cuda.current_stream()
        for _ in range(2):                                  # second call reuses the registered buffer
            b1, m1 = F.fbspca_covariance(plan, coeffs, coeffs.shape[1], coeffs.shape[1], comm, stream=stream)
            F.fbspca_comm_wait(comm, stream, timeout_s=30.0)
            assert torch.equal(b0, b1) and torch.equal(m0, m1)
        # the stand-alone all-reduce on a caller buffer, and the streaming (accumulate) form
        part = F.fbspca_covariance_partial(plan, coeffs)
        ref = part.clone()
        F.fbspca_allreduce_partial(plan, part, comm)
        F.fbspca_comm_wait(comm, stream, timeout_s=30.0)
        assert torch.equal(part, ref)
    finally:
        F.fbspca_comm_destroy(comm)


@pytest.mark.parametrize("with_comm", [False, True])
def test_step_graph_replay_equals_eager(c2, with_comm):
    """fbspca_step: eager, then captured (expand + both K5 streams + all-reduce + finalise in one CUDA graph),
    then replayed -- every result identical to the eager call, for new data in the same buffers too."""
    plan, imgs, _ = c2
    n = imgs.shape[0]
    comm = F.fbspca_comm_init(F.fbspca_nccl_unique_id(), 1, 0) if with_comm else None
    try:
        s = torch.cuda.Stream()
        coeffs = torch.empty((plan.n_coef, n), dtype=plan.complex_dtype, device=DEV)
        blocks = torch.empty(plan.n_blk, dtype=torch.float64, device=DEV)
        mean = torch.empty(int(plan.p[0]), dtype=torch.float64, device=DEV)
        with torch.cuda.stream(s):
            src = imgs.clone()
            F.fbspca_step(plan, src, coeffs, blocks, mean, n, comm, use_graph=False, stream=s)
            eager_b, eager_m = blocks.clone(), mean.clone()
            for _ in range(3):                             # eager (first), capture + launch, replay
                blocks.zero_(); mean.zero_()
                F.fbspca_step(plan, src, coeffs, blocks, mean, n, comm, use_graph=True, stream=s)
                torch.cuda.synchronize()
                assert torch.equal(blocks, eager_b) and torch.equal(mean, eager_m)
            src.mul_(2.0)                                  # new data in the captured buffers: scaled 4x / 2x
            F.fbspca_step(plan, src, coeffs, blocks, mean, n, comm, use_graph=True, stream=s)
            torch.cuda.synchronize()
        assert torch.allclose(blocks, 4 * eager_b, rtol=1e-5, atol=1e-9)
        assert torch.allclose(mean, 2 * eager_m, rtol=1e-5, atol=1e-9)
    finally:
        if comm:
            F.fbspca_comm_destroy(comm)


def test_plan_on_second_thread_gets_smem_optin(c2):
    """The shared-memory opt-in is recorded per (kernel, device): a plan used from another host thread launches."""
    import threading
    plan, imgs, coeffs = c2
    out = {}

    def run():
        try:
            p2 = F.fbspca_plan(plan.L, plan.c, plan.R, device=0, max_batch=256)
            c = F.fbspca_expand(p2, imgs[:300])
            torch.cuda.synchronize()
            out["diff"] = ((c - coeffs[:, :300]).abs().max() / coeffs[:, :300].abs().max()).item()
        except Exception as e:                              # pragma: no cover
            out["err"] = repr(e)
    t = threading.Thread(target=run)
    t.start(); t.join()
    assert "err" not in out, out.get("err")
    assert out["diff"] <= 1e-6
