"""CPU tests of the row-strip sharding host logic: layout arithmetic and the
neighbour exchange over a real torch.distributed group (gloo, world size 2)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1901_06110_b200.parallel import LocalComm, StripLayout, TorchComm


@pytest.mark.parametrize("H,W,R,P,N", [(8192, 8192, 10, 7, 8), (8192, 8192, 10, 7, 3),
                                       (300, 100, 10, 7, 2), (1000, 64, 21, 3, 4)])
def test_layout_partitions_tile_rows(H, W, R, P, N):
    lays = [StripLayout(H, W, R, P, N, r) for r in range(N)]
    for lay in lays:
        lay.validate()
    assert lays[0].tile_rows[0] == 0 and lays[-1].tile_rows[1] == lays[0].tiles_y
    for a, b in zip(lays, lays[1:]):
        assert a.tile_rows[1] == b.tile_rows[0]
        assert a.rows[1] == b.rows[0]
        assert a.rows[1] % a.TH == 0
    assert lays[-1].rows[1] == H
    p = (P - 1) // 2
    for lay in lays:
        b0, b1 = lay.window
        y0, y1 = lay.rows
        assert b0 == max(0, y0 - p) and b1 == min(H, y1 + R + max(p, 4))
        first, off, nslot = lay.part
        assert first == max(0, lay.tile_rows[0] - lay.dti)
        assert nslot - off == lay.tile_rows[1] - lay.tile_rows[0]


def test_layout_rejects_thin_strips():
    with pytest.raises(ValueError):
        for r in range(8):
            StripLayout(100, 64, 10, 7, 8, r).validate()


class _S:
    def __init__(self, rank):
        self.t = torch.full((6,), float(rank))
        self.mbits = torch.tensor([rank * 10 + 3], dtype=torch.int32)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchComm()
        st = _S(rank)
        # down: my last 2 -> next rank's first 2 ; up: my [2:4] -> prev rank's [4:6]
        comm.shift_down([st], lambda s: s.t[4:6], lambda s: s.t[0:2])
        comm.shift_up([st], lambda s: s.t[2:4], lambda s: s.t[4:6])
        comm.allreduce_max([st])
        # index-addressed shifts and the sum all-reduce used by ShardedSRADMM
        buf = [torch.arange(4, dtype=torch.float64) + 10 * rank]
        comm.shift(world, lambda k: buf[0][2:4], lambda k: buf[0][0:2], +1)
        comm.shift(world, lambda k: buf[0][0:1], lambda k: buf[0][3:4], -1)
        tot = torch.tensor([1.5 * (rank + 1), float(rank)], dtype=torch.float64)
        comm.allreduce_sum([tot])
        # deferred completion: post, do unrelated work, then finish
        st2 = _S(rank + 5)
        fin = comm.start_shift([st2], lambda s: s.t[4:6], lambda s: s.t[0:2], +1)
        st2.t[2:4] += 100.0
        fin()
        tot = torch.cat([tot, st2.t.to(torch.float64)])
        q.put((rank, st.t.tolist(), int(st.mbits[0]), buf[0].tolist(), tot.tolist()))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_torch_comm_gloo_world2_matches_local():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (t, m, b, s)) for r, t, m, b, s in (q.get(timeout=120) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # the same exchanges with the in-process communicator
    states = [_S(r) for r in range(world)]
    comm = LocalComm()
    comm.shift_down(states, lambda s: s.t[4:6], lambda s: s.t[0:2])
    comm.shift_up(states, lambda s: s.t[2:4], lambda s: s.t[4:6])
    comm.allreduce_max(states)
    for r in range(world):
        assert res[r][0] == states[r].t.tolist()
        assert res[r][1] == int(states[r].mbits[0]) == 13
    assert res[0][0] == [0, 0, 0, 0, 1, 1] and res[1][0] == [0, 0, 1, 1, 1, 1]
    bufs = [torch.arange(4, dtype=torch.float64) + 10 * r for r in range(world)]
    comm.shift(world, lambda k: bufs[k][2:4], lambda k: bufs[k][0:2], +1)
    comm.shift(world, lambda k: bufs[k][0:1], lambda k: bufs[k][3:4], -1)
    tots = [torch.tensor([1.5 * (r + 1), float(r)], dtype=torch.float64) for r in range(world)]
    comm.allreduce_sum(tots)
    st2 = [_S(r + 5) for r in range(world)]
    fin = comm.start_shift(st2, lambda s: s.t[4:6], lambda s: s.t[0:2], +1)
    for s_ in st2:
        s_.t[2:4] += 100.0
    fin()
    tots = [torch.cat([tots[r], st2[r].t.to(torch.float64)]) for r in range(world)]
    for r in range(world):
        assert res[r][2] == bufs[r].tolist()
        assert res[r][3] == tots[r].tolist()
        assert res[r][3][:2] == [4.5, 1.0]
    assert res[1][3][2:] == [5, 5, 106, 106, 6, 6] and res[0][3][2:] == [5, 5, 105, 105, 5, 5]
    assert bufs[0].tolist() == [0, 1, 2, 2] and bufs[1].tolist() == [2, 3, 12, 13]
