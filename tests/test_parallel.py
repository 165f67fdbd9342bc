"""Multi-process (world_size 2, gloo, CPU) tests of the batch-sharded data-parallel path.

Each rank runs the FP64 oracle on its batch shard (standing in for libce on a
GPU); the all-reduced factor gradients and the gathered outputs / X gradients
must equal a single-process full-batch run exactly (up to FP64 summation order).
"""
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2401_03384_b200.parallel import allreduce_factor_grads, data_parallel_step, shard_range


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_covers_batch():
    for b in (1, 2, 7, 128, 1024):
        for w in (1, 2, 3, 4, 8):
            spans = [shard_range(b, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == b
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def _layer():
    import paper_2401_03384_b200 as ce
    le = ce.expression(ce.LayerSpec("cp", [6], [5], 3, 3, 6, 6, 4, [3]))
    plan = ce.optimal(le.expr, le.dims, "same", "training")
    nodes = [(n["left"], n["right"], n["result"]) for n in json.loads(plan.to_json())["nodes"]]
    return le, nodes


def _oracle_fwd_bwd(le, nodes):
    from oracle import np_oracle as npo

    def f(xs, dy):
        dims = [list(x.shape) for x in xs]
        ins = [x.numpy() for x in xs]
        out, _ = npo.execute(le.expr, dims, nodes, ins)
        grads = npo.backward(le.expr, dims, nodes, ins, dy.numpy())
        return torch.from_numpy(out), [torch.from_numpy(np.ascontiguousarray(g)) for g in grads]
    return f


def _worker(rank, world, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    le, nodes = _layer()
    from oracle import np_oracle as npo
    xs = [torch.from_numpy(npo.fill_random(d, 1000 + i)) for i, d in enumerate(le.dims)]
    import paper_2401_03384_b200 as ce
    plan = ce.optimal(le.expr, le.dims, "same", "training")
    dy = torch.from_numpy(npo.fill_random(plan.out_dims, 2000))
    out, grads = data_parallel_step(xs, dy, rank, world, _oracle_fwd_bwd(le, nodes))
    result_q.put((rank, out.numpy(), [g.numpy() for g in grads]))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_matches_full_batch():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process reference
    le, nodes = _layer()
    from oracle import np_oracle as npo
    xs = [torch.from_numpy(npo.fill_random(d, 1000 + i)) for i, d in enumerate(le.dims)]
    import paper_2401_03384_b200 as ce
    plan = ce.optimal(le.expr, le.dims, "same", "training")
    dy = torch.from_numpy(npo.fill_random(plan.out_dims, 2000))
    out, grads = _oracle_fwd_bwd(le, nodes)(xs, dy)
    np.testing.assert_allclose(np.concatenate([r[1] for r in res]), out.numpy(), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(np.concatenate([r[2][0] for r in res]), grads[0].numpy(), rtol=1e-12, atol=1e-12)
    for i in range(1, len(grads)):
        for r in res:  # every rank holds the full (all-reduced) factor gradient
            np.testing.assert_allclose(r[2][i], grads[i].numpy(), rtol=1e-10, atol=1e-12)


def _async_worker(rank, world, port, result_q):
    import os
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2401_03384_b200.parallel import allreduce_factor_grads_async
    grads = [torch.full((3,), float(rank)), torch.arange(4.0) * (rank + 1), None, torch.ones(2, 2) * rank]
    out, work = allreduce_factor_grads_async(grads)
    assert work is not None
    work.wait()
    result_q.put((rank, [None if g is None else g.numpy() for g in out]))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_async_allreduce():
    """Asynchronous bucketed factor-gradient all-reduce (bench.py overlaps it with the next
    layer): X (index 0) untouched, every factor gradient summed over the ranks."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_async_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, g in res:
        np.testing.assert_array_equal(g[0], np.full(3, float(rank)))
        np.testing.assert_array_equal(g[1], np.arange(4.0) * 3)
        assert g[2] is None
        np.testing.assert_array_equal(g[3], np.ones((2, 2)))


def test_allreduce_is_identity_without_process_group():
    g = [torch.ones(3), torch.ones(2)]
    out = allreduce_factor_grads(g)
    assert all(torch.equal(a, b) for a, b in zip(out, g))
