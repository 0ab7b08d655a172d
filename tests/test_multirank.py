"""N>1 host logic on CPU: world_size-2 gloo process group.  Each rank takes its
pixel block of one frame (paper_2203_00952_b200.shard), computes the oracle
sketch + gradient of its block, and the gathered result must equal the
full-frame computation exactly (pixels are independent: no data-path
collective).  Also checks the bench's max-over-ranks timing reduction."""
import os
import socket
import sys

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import oracle
    import srt3d_inputs
    from paper_2203_00952_b200.shard import pixel_range, shard_csr

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    f = srt3d_inputs.make_frame("C3", rows=12, cols=10)
    i0, i1 = pixel_range(f.npix, world, rank)
    b, o = shard_csr(f.bins, f.offsets, i0, i1)
    z = oracle.sketch(b, o, f.T, f.m)
    t0, a0 = f.theta0()
    gt, ga, L = oracle.sketch_grad(z, t0[i0:i1], a0[i0:i1], f.sigma, f.T, f.m)
    local = torch.from_numpy(np.concatenate([z.real, z.imag, gt, ga, L[:, None]], axis=1))
    sizes = [None] * world
    dist.all_gather_object(sizes, local.shape[0])
    buf = [torch.zeros((n, local.shape[1]), dtype=local.dtype) for n in sizes]
    dist.all_gather(buf, local)
    # bench-style timing reduction: max over ranks
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put((torch.cat(buf).numpy(), float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_equal_full_frame():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sys.path.insert(0, ROOT)
    import oracle
    import srt3d_inputs

    f = srt3d_inputs.make_frame("C3", rows=12, cols=10)
    z = oracle.sketch(f.bins, f.offsets, f.T, f.m)
    t0, a0 = f.theta0()
    gt, ga, L = oracle.sketch_grad(z, t0, a0, f.sigma, f.T, f.m)
    full = np.concatenate([z.real, z.imag, gt, ga, L[:, None]], axis=1)
    assert np.array_equal(got, full)
    assert tmax == 2.0


def test_pixel_range_partition():
    from paper_2203_00952_b200.shard import pixel_range

    for npix in (0, 1, 7, 262144, 1001):
        for world in (1, 2, 3, 8):
            r = [pixel_range(npix, world, k) for k in range(world)]
            assert r[0][0] == 0 and r[-1][1] == npix
            assert all(r[k][1] == r[k + 1][0] for k in range(world - 1))
            sizes = [b - a for a, b in r]
            assert max(sizes) - min(sizes) <= 1
