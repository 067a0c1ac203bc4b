"""The host-staged communicator's transport (lrcnn.Comm.host) on CPU: two gloo processes call the
exchange / all-reduce callbacks exactly as liblrcnn.so does (C arrays of peers, send flags, host
pointers and byte counts) and must move the bytes of the halo schedule the planner produced for
their rank (lrcnn_plan_xfers) and sum the gradients.  The device side (staging copies) runs in
tests/test_gpu_dist_host.py."""
import ctypes
import os
import socket
import tempfile

import numpy as np
import pytest

import workloads as WL

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist
    from paper_2401_11471_b200 import lrcnn as LB
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=rank, world_size=world)
    comm = LB.Comm.host()
    exchange, allreduce = comm._callbacks
    # the halo schedule of segment 1 of a row-sharded VGG (as the library would stage it)
    net = WL.vgg16(H=64, W=32, width_div=8, segments="pool")
    plan = LB.Plan(net, 2, mode="2ps", prec="bf16", world=world, rank=rank, n_bands=2)
    xs = plan.xfers(1)
    n = len(xs)
    bufs, ptrs = [], (ctypes.c_void_p * n)()
    for i, (peer, send, r0, r1) in enumerate(xs):
        nbytes = (r1 - r0) * 1000 + 7
        b = np.zeros(nbytes, dtype=np.uint8)
        if send:   # payload identifies (sender, receiver, rows)
            b[:] = (np.arange(nbytes) * 7 + 31 * rank + 5 * peer + r0) % 251
        bufs.append(b)
        ptrs[i] = b.ctypes.data
    peers = (ctypes.c_int * n)(*[x[0] for x in xs])
    sends = (ctypes.c_int * n)(*[x[1] for x in xs])
    sizes = (ctypes.c_size_t * n)(*[b.size for b in bufs])
    rc = exchange(None, n, peers, sends, ptrs, sizes)
    g = np.arange(1000, dtype=np.float32) * (rank + 1)
    rc2 = allreduce(None, g.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), g.size)
    np.savez(os.path.join(out_dir, "r%d.npz" % rank), rc=rc, rc2=rc2, g=g,
             recv=np.array([i for i, x in enumerate(xs) if not x[1]]), xs=np.array(xs),
             **{"b%d" % i: b for i, b in enumerate(bufs)})
    comm.free()
    dist.destroy_process_group()


def test_host_comm_callbacks_two_processes():
    import torch.multiprocessing as mp
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        res = [dict(np.load(os.path.join(d, "r%d.npz" % r))) for r in range(world)]
    for rank, r in enumerate(res):
        assert int(r["rc"]) == 0 and int(r["rc2"]) == 0
        assert np.array_equal(r["g"], np.arange(1000, dtype=np.float32) * 3)      # 1x + 2x
        assert len(r["xs"]) > 0
        for i in r["recv"]:
            peer, send, r0, r1 = r["xs"][i]
            nbytes = (r1 - r0) * 1000 + 7
            want = (np.arange(nbytes) * 7 + 31 * peer + 5 * rank + r0) % 251
            assert np.array_equal(r["b%d" % i], want.astype(np.uint8)), (rank, i)
