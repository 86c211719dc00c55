"""Multi-rank mask sharding (evaluate_distributed) on the CPU with gloo.

Each rank owns partition_columns(2^m - 1, world)[rank] (parallel.py:38-57);
the exchange is one all-reduce(MAX) of the packed (max|W|, ~v) key plus one
all-gather of the padded per-component NL shards.  The per-shard compute is
injected (the oracle) so the exchange runs here without a GPU; on a GPU box
the default compute is libsbw (covered in test_gpu_parity.py).
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_shard(s, lo, hi):
    from oracle import sbw_oracle as orc

    mx = orc.component_max_abs(s.table, s.n, lo, hi)
    i = int(np.argmax(mx))  # first = smallest v among the maxima
    key = (int(mx[i]) << 32) | (0xFFFFFFFF - (lo + i))
    return ((1 << s.n) - mx) >> 1, key


def _worker(rank, world, port, n, m, seed, bij, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1912_03732_b200 as sw

        s = sw.generate_sbox(n, m, seed, bijective=bij)
        res, cm = sw.evaluate_distributed(s, compute=_oracle_shard)
        q.put((rank, res.value, res.argmin_v, cm.values.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,m,seed,bij", [(2, 8, 8, 0, True), (3, 9, 5, 4, False),
                                                (2, 7, 1, 2, False), (4, 6, 2, 1, False)])
def test_sharded_nl_equals_single_process(world, n, m, seed, bij):
    from oracle import sbw_oracle as orc

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, m, seed, bij, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    t = orc.gen_table(n, m, seed, bij)
    want = orc.component_nl(t, n, 1, 1 << m)
    wv, wa = orc.nl_from_maxima(want)
    for rank, value, argmin, values in out:
        assert (value, argmin) == (wv, wa), rank
        assert np.array_equal(np.array(values), want), rank


# ---------------------------------------------------------------------------
# spectrum_distributed: the materialised Walsh matrix sharded over the ranks
# ---------------------------------------------------------------------------
def _oracle_spectrum_shard(s, lo, hi, layout):
    from oracle import sbw_oracle as orc

    rows = orc.spectrum(s.table, s.n, lo, hi)
    mx = np.abs(rows).max(axis=1).astype(np.int32)
    return (rows if layout == "mask" else rows.T), mx


def _spec_worker(rank, world, port, n, m, seed, bij, layout, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1912_03732_b200 as sw

        s = sw.generate_sbox(n, m, seed, bijective=bij)
        shard, (lo, hi), res = sw.spectrum_distributed(s, layout=layout, compute=_oracle_spectrum_shard)
        q.put((rank, lo, hi, res.value, res.argmin_v, shard.numpy().tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,m,seed,bij,layout", [(2, 8, 8, 0, True, "mask"), (3, 7, 5, 4, False, "x"),
                                                       (4, 6, 2, 1, False, "mask"), (2, 5, 3, 2, False, "x")])
def test_sharded_spectrum_equals_single_process(world, n, m, seed, bij, layout):
    """Each rank holds exactly its partition_columns range of the matrix in
    the requested layout; the shards tile the whole matrix; every rank gets
    the global NL from the one key all-reduce.  (m = 2 with world 4 leaves
    rank 3 an empty shard.)"""
    from oracle import sbw_oracle as orc

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_spec_worker, args=(r, world, port, n, m, seed, bij, layout, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    t = orc.gen_table(n, m, seed, bij)
    full = orc.spectrum(t, n, 1, 1 << m)
    wv, wa = orc.nl_from_maxima(orc.component_nl(t, n, 1, 1 << m))
    want_ranges = list(orc.partition_columns((1 << m) - 1, world))
    want_ranges += [((1 << m), (1 << m))] * (world - len(want_ranges))
    for rank, lo, hi, value, argmin, shard in out:
        assert (lo, hi) == tuple(want_ranges[rank])
        assert (value, argmin) == (wv, wa), rank
        want = full[lo - 1:hi - 1]
        got = np.asarray(shard, dtype=np.int32).reshape((hi - lo, 1 << n) if layout == "mask" else (1 << n, hi - lo))
        assert np.array_equal(got, want if layout == "mask" else want.T), rank
