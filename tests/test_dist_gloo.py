"""Multi-process host logic of the z-slab sharding (paper_2509_25044_b200.dist) on CPU
with the gloo backend, world sizes 2 and 3 (the transport the B200 path runs over NCCL).
Reference semantics: fabric.hpp:31-370, distops.hpp:36-49."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_25044_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # surface worker failures to the parent
        q.put((rank, e))
    finally:
        dist.destroy_process_group()


def spawn(fn, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_run, args=(r, world, port, fn, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    for r, v in out.items():
        if isinstance(v, Exception):
            raise v
    return out


def volume(shape, seed=0):
    g = np.random.default_rng(seed)
    return torch.from_numpy(g.random(shape).astype(np.float32))


# ---- workers (module level: picklable for spawn) --------------------------------
def w_halo(rank, world):
    shape = (11, 4, 5)
    v = volume(shape)
    spec = D.make_shard_spec(shape, world, rank)
    out, lo, hi = D.halo_exchange(v[spec.lo:spec.hi].clone(), spec, 3)
    z0 = spec.lo - lo
    ok = torch.equal(out, v[z0:z0 + out.shape[0]])
    return ok, lo, hi


def w_fetch(rank, world):
    shape = (13, 3, 4)
    v = volume(shape, 1)
    spec = D.make_shard_spec(shape, world, rank)
    # every rank asks for a different window, some spanning several owners
    z0, z1 = [(0, 13), (2, 9), (5, 13)][rank % 3]
    got = D.fetch_planes(v[spec.lo:spec.hi].clone(), spec, z0, z1)
    return torch.equal(got, v[z0:z1])


def w_allreduce(rank, world):
    t = torch.arange(6, dtype=torch.float64) * (rank + 1)
    a = D.allreduce_sum(t.clone())
    b = D.allreduce_sum(t.clone(), ordered=True)
    ref = torch.arange(6, dtype=torch.float64) * sum(r + 1 for r in range(world))
    return torch.equal(a, ref) and torch.equal(b, ref)


def w_halo_too_thick(rank, world):
    shape = (5, 2, 2)
    spec = D.make_shard_spec(shape, world, rank)
    try:
        D.halo_exchange(torch.zeros(spec.local_shape), spec, 3)
    except ValueError as e:
        return "exceeds" in str(e)
    return False


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_matches_unsharded(world):
    out = spawn(w_halo, world)
    for r in range(world):
        ok, lo, hi = out[r]
        assert ok
        assert lo == (3 if r > 0 else 0) and hi == (3 if r < world - 1 else 0)


@pytest.mark.parametrize("world", [2, 3])
def test_fetch_planes_gathers_any_window(world):
    assert all(spawn(w_fetch, world).values())


def test_allreduce_plain_and_rank_ordered():
    assert all(spawn(w_allreduce, 3).values())


def test_halo_rejects_pad_thicker_than_neighbour():
    assert all(spawn(w_halo_too_thick, 3).values())


# ---- single-process rules ----------------------------------------------------------
def test_shard_ranges_and_specs(orc):
    for n, w in [(10, 3), (256, 8), (7, 7), (1200, 8)]:
        rs = D.shard_ranges(n, w)
        assert rs == [orc.shard_range(n, w, r) for r in range(w)]
        assert rs[0][0] == 0 and rs[-1][1] == n
    with pytest.raises(ValueError):
        D.shard_ranges(2, 3)
    s = D.make_shard_spec((10, 4, 4), 3, 1)
    assert (s.lo, s.hi) == (4, 7)
    assert s.x_min[2] == pytest.approx(-1 + 2 * 4 / 9) and s.x_max[2] == pytest.approx(-1 + 2 * 6 / 9)


def test_shard_rescale_solves_boundary_conditions():
    s = D.make_shard_spec((9, 4, 4), 2, 1)
    rs = D.compute_shard_rescale(s.x_min, s.x_max)
    for c in range(3):  # distops.hpp:34-35 (test_distops.cpp:125-137)
        assert rs.S[c] * s.x_min[c] + rs.t[c] == pytest.approx(-1.0)
        assert rs.S[c] * s.x_max[c] + rs.t[c] == pytest.approx(1.0)
