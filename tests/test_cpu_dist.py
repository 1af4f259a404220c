"""World-size-2 gloo test of the multi-GPU plumbing on CPU: clips sharded per
rank, per-rank kernel gradients (computed here by the CPU oracle as a stand-in
for the device GEMMs), one flattened all-reduce -> equals the full-batch
gradient."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import spectro_oracle as O
    from paper_1912_12055_b200.dist import allreduce_grads, gather_shards, shard_batch
    rng = np.random.default_rng(0)
    x = torch.from_numpy((rng.standard_normal((5, 800)) * 0.5).astype(np.float32))
    g = rng.standard_normal((5, 33, 800 // 16 + 1))
    h_re, h_im = O.stft_bank(64, 8000.0)
    mine = shard_batch(x, rank, world)
    lo = sum(shard_batch(x, r, world).shape[0] for r in range(rank))
    p_re = torch.nn.Parameter(torch.zeros(h_re.shape, dtype=torch.float64))
    p_im = torch.nn.Parameter(torch.zeros(h_im.shape, dtype=torch.float64))
    p_re.grad = torch.zeros_like(p_re)
    p_im.grad = torch.zeros_like(p_im)
    for i, c in enumerate(mine.numpy()):
        gr = O.conv_layer_vjp(c.astype(np.float64), h_re, h_im, 16, g[lo + i])
        p_re.grad += torch.from_numpy(gr["h_re"])
        p_im.grad += torch.from_numpy(gr["h_im"])
    allreduce_grads([p_re, p_im])
    S = torch.from_numpy(np.stack([O.smooth_mag_forward(c.astype(np.float64), h_re, h_im, 16)[3]
                                   for c in mine.numpy()]))
    full = gather_shards(S, 5)
    if rank == 0:
        torch.save({"re": p_re.grad, "im": p_im.grad, "S": full}, out_path)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_grad_allreduce(tmp_path):
    out = str(tmp_path / "r0.pt")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    from oracle import spectro_oracle as O
    res = torch.load(out)
    rng = np.random.default_rng(0)
    x = (rng.standard_normal((5, 800)) * 0.5).astype(np.float32)
    g = rng.standard_normal((5, 33, 800 // 16 + 1))
    h_re, h_im = O.stft_bank(64, 8000.0)
    ref_re = sum(O.conv_layer_vjp(x[i].astype(np.float64), h_re, h_im, 16, g[i])["h_re"] for i in range(5))
    ref_im = sum(O.conv_layer_vjp(x[i].astype(np.float64), h_re, h_im, 16, g[i])["h_im"] for i in range(5))
    assert np.allclose(res["re"].numpy(), ref_re, rtol=1e-12, atol=1e-9)
    assert np.allclose(res["im"].numpy(), ref_im, rtol=1e-12, atol=1e-9)
    S = np.stack([O.smooth_mag_forward(c.astype(np.float64), h_re, h_im, 16)[3] for c in x])
    assert np.array_equal(res["S"].numpy(), S)


class _FakeOp:
    """Stands in for autograd.DftLayerOp: a backward that finishes gradient
    blocks in the device order (mel weights, dK rows [0, 1024), the rest) and
    hands each to the armed reducer, then waits before returning."""

    reducer = None

    def backward(self, rank):
        g = torch.Generator().manual_seed(100 + rank)
        dW = torch.randn(128, 1025, generator=g, dtype=torch.float64)
        dk = torch.randn(2050, 64, generator=g, dtype=torch.float64)
        self.reducer.launch(dW)
        for r0, r1 in [(0, 1024), (1024, 2050)]:
            self.reducer.launch(dk[r0:r1])
        self.reducer.wait()
        return dW, dk


def _reducer_worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1912_12055_b200.dist import GradReducer
    op = _FakeOp()
    red = GradReducer([op])
    for step in range(2):  # re-armed every step
        red.arm()
        assert op.reducer is red
        dW, dk = op.backward(rank)
        red.finish()
        assert op.reducer is None and red.buckets == 3
    if rank == 0:
        torch.save({"dW": dW, "dk": dk}, out_path)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_bucketed_reducer(tmp_path):
    """dist.GradReducer (the bucketed, overlapped gradient all-reduce of the
    trainable layers) on world-size-2 gloo: every bucket equals the sum over ranks."""
    out = str(tmp_path / "red.pt")
    mp.spawn(_reducer_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    res = torch.load(out)
    want_W = sum(_FakeOp.__dict__["backward"].__get__(_Stub())(r)[0] for r in range(2))
    want_k = sum(_FakeOp.__dict__["backward"].__get__(_Stub())(r)[1] for r in range(2))
    assert torch.equal(res["dW"], want_W)
    assert torch.equal(res["dk"], want_k)


class _Stub:
    class reducer:  # local (no process group): launch / wait are no-ops
        @staticmethod
        def launch(t):
            pass

        @staticmethod
        def wait():
            pass
