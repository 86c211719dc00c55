"""evaluate_distributed(transport="p2p"): the shards' maxima and keys are
written into rank 0's device memory through CUDA IPC mappings (sbw_ipc_*,
sbw_key_merge, include/sbw.h) -- no collective on the data path.

gpurun offers one GPU, so the ranks here share cuda:0: the IPC mapping,
the kernels' stores into another process's allocation, the system-scope key
atomics and the peer read-back are the same code path as across NVLink; the
ranks' kernels never wait on one another (only host barriers on gloo).
Results must equal the single-process evaluation and the oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, m, seed, bij, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1912_03732_b200 as sw

        s = sw.generate_sbox(n, m, seed, bijective=bij)
        res, cm = sw.evaluate_distributed(s, transport="p2p")
        q.put((rank, res.value, res.argmin_v, cm.values.tolist()))
    except Exception as e:  # surface the failure to the parent
        q.put((rank, None, None, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,m,seed,bij", [(2, 12, 12, 0, True),    # K2 tensor-core NL
                                                (3, 9, 7, 4, False),     # K1 / K0, uneven shards
                                                (2, 17, 9, 5, False)])   # K3 multi-pass (+ scratch)
def test_p2p_sharded_nl_equals_single_process(world, n, m, seed, bij):
    import paper_1912_03732_b200 as sw
    from oracle import sbw_oracle as orc

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, m, seed, bij, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(o[1] is not None for o in out), out
    s = sw.generate_sbox(n, m, seed, bijective=bij)
    _, cm = sw.fwht_fused(s, mode="stream")
    want = sw.nonlinearity_from_maxima(cm)
    for rank, value, argmin, values in out:
        assert (value, argmin) == (want.value, want.argmin_v), rank
        assert np.array_equal(np.asarray(values), cm.values), rank
    lo, hi = 1, min(1 << m, 65)
    assert np.array_equal(cm.values[: hi - lo], orc.component_nl(s.table, n, lo, hi))


def _spec_worker(rank, world, port, n, m, seed, bij, layout, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import hashlib

        import paper_1912_03732_b200 as sw

        s = sw.generate_sbox(n, m, seed, bijective=bij)
        shard, (lo, hi), res = sw.spectrum_distributed(s, layout=layout)
        assert shard.is_cuda
        h = hashlib.sha256(shard.cpu().numpy().tobytes()).hexdigest()
        q.put((rank, lo, hi, res.value, res.argmin_v, h))
    except Exception as e:
        q.put((rank, None, None, None, None, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,m,seed,bij,layout", [(2, 12, 12, 0, True, "mask"),   # K2 spectrum
                                                       (3, 13, 9, 3, False, "x"),      # K2 + transpose
                                                       (2, 17, 6, 5, False, "mask")])  # K3 spectrum
def test_sharded_spectrum_on_gpu(world, n, m, seed, bij, layout):
    """spectrum_distributed with libsbw: each rank's device shard equals its
    range of the single-process matrix (in the requested layout) and of the
    oracle; the global NL comes from the one key all-reduce."""
    import hashlib

    import paper_1912_03732_b200 as sw
    from oracle import sbw_oracle as orc

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_spec_worker, args=(r, world, port, n, m, seed, bij, layout, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(o[1] is not None for o in out), out
    s = sw.generate_sbox(n, m, seed, bijective=bij)
    full = orc.spectrum(s.table, n, 1, 1 << m)
    want = orc.nl_from_maxima(orc.component_nl(s.table, n, 1, 1 << m))
    for rank, lo, hi, value, argmin, h in out:
        assert (value, argmin) == want, rank
        part = full[lo - 1:hi - 1]
        ref = np.ascontiguousarray(part if layout == "mask" else part.T)
        assert h == hashlib.sha256(ref.tobytes()).hexdigest(), rank
