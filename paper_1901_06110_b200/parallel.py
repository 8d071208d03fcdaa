"""Row-strip sharding of DSG-NLM across GPUs.

A large image (config 4: 8192^2) is split into row strips of whole tiles,
one per rank (one process per GPU, ``torch.distributed`` over NCCL for the
plumbing).  One adaptive denoise is

    halo rows of the input (pnp_dsg_geometry: p above,
      R + max(p, KY) below for the P-templated sweep)        [P2P exchange]
    sweep A (mass g) on own tile rows (+ the strip's k cache when it fits)
    the last ceil(R/TH) tile rows of partial blocks -> next rank
    fixup: rs = g^-1/2 on own rows
    the rs rows the sweep reads below -> previous rank       [P2P exchange]
    sweep B (K x and d) on own tile rows (streams the k cache if present)
    partial blocks -> next rank                                [P2P exchange]
    fixup: K x, d, local max d
    all-reduce max -> m (the north-star "alpha")               [NCCL max]
    finalize own rows: W x = K x / m + (1 - d/m) x

Strip boundaries sit on tile boundaries and every rank sums each pixel's
contributions in the single-GPU order, so the sharded output is
bit-identical to one GPU.  The algorithm is written once over a list of
per-rank states and a communicator: ``TorchComm`` moves data between real
ranks (NCCL / gloo), ``LocalComm`` runs N virtual ranks in one process on
one device (test / development mode; copies instead of messages).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import torch

from . import _lib as L
from .denoise import PatchParams

@dataclass(frozen=True)
class StripLayout:
    """Which rows / tile rows rank ``rank`` of ``nranks`` owns and reads.
    Tile height, block band and halos come from the library
    (``pnp_dsg_geometry``): they depend on the sweep path, i.e. on (R, P)
    and whether the patch taps are the reference's box taps."""

    Hg: int
    W: int
    R: int
    P: int
    nranks: int
    rank: int
    box: bool = False

    @property
    def geom(self) -> tuple:
        return L.dsg_geometry(self.Hg, self.W, self.R, self.P, self.box)

    @property
    def TH(self) -> int:
        return self.geom[0]

    @property
    def Rb(self) -> int:
        """Far band of a partial block (0: blocks cover the tile only)."""
        return self.geom[2]

    @property
    def rs_below(self) -> int:
        """Rows of the channel planes a tile row's sweep reads below it."""
        return self.geom[6]

    @property
    def tiles_y(self) -> int:
        return -(-self.Hg // self.TH)

    @property
    def tile_rows(self) -> tuple[int, int]:
        t = self.tiles_y
        return (self.rank * t) // self.nranks, ((self.rank + 1) * t) // self.nranks

    @property
    def rows(self) -> tuple[int, int]:
        t0, t1 = self.tile_rows
        return t0 * self.TH, min(t1 * self.TH, self.Hg)

    @property
    def dti(self) -> int:
        """Tile rows of the rank above whose partial blocks reach our rows."""
        return -(-self.Rb // self.TH)

    @property
    def halo(self) -> tuple[int, int]:
        g = self.geom
        return g[4], g[5]

    @property
    def window(self) -> tuple[int, int]:
        """Rows [b0, b1) held locally: own rows plus halos, clipped to the image."""
        y0, y1 = self.rows
        top, bot = self.halo
        return max(0, y0 - top), min(self.Hg, y1 + bot)

    @property
    def part(self) -> tuple[int, int, int]:
        """(global tile row of slot 0, slot of our first tile row, slots)."""
        t0, t1 = self.tile_rows
        first = max(0, t0 - self.dti)
        return first, t0 - first, t1 - first

    def validate(self) -> None:
        t0, t1 = self.tile_rows
        if t1 - t0 < max(self.dti, 1):
            raise ValueError("strip too thin: each rank needs >= ceil(R/TH) tile rows")
        y0, y1 = self.rows
        if y1 - y0 < self.halo[1] and self.rank < self.nranks - 1:
            raise ValueError("strip too thin for the halo")


class _RankState:
    """Device buffers of one rank (or one virtual rank)."""

    def __init__(self, lay: StripLayout, device):
        self.lay = lay
        b0, b1 = lay.window
        self.buf = torch.zeros((b1 - b0, lay.W), dtype=torch.float32, device=device)
        self.rs = torch.zeros_like(self.buf)
        self.kx = torch.zeros_like(self.buf)
        self.d = torch.zeros_like(self.buf)
        self.out = torch.zeros_like(self.buf)
        self.mbits = torch.zeros(1, dtype=torch.int32, device=device)
        box = int(lay.box)
        pf = int(L.lib.pnp_dsg_partial_floats(lay.Hg, lay.W, lay.R, lay.P, box, 2, lay.part[2]))
        if pf < 0:
            raise ValueError(L.lib.pnp_last_error().decode())
        self.partial = torch.zeros(pf, dtype=torch.float32, device=device)
        self.block_floats_c1 = int(L.lib.pnp_dsg_partial_floats(lay.Hg, lay.W, lay.R, lay.P, box,
                                                                1, 1))
        self.block_floats_c2 = 2 * self.block_floats_c1
        self.kcache = None
        self.kc_per_tile_row = 0

    def enable_kcache(self, headroom: int = 4 << 30) -> bool:
        """Keep this strip's pair weights in HBM (sweep A stores, sweep B
        streams them: bitwise neutral) when they fit with ``headroom`` spare."""
        lay = self.lay
        t0, t1 = lay.tile_rows
        n = int(L.lib.pnp_dsg_kcache_floats(lay.Hg, lay.W, lay.R, lay.P, int(lay.box), t1 - t0))
        free, _ = torch.cuda.mem_get_info(self.buf.device)
        if n <= 0 or 4 * n + headroom > free:
            return False
        self.kcache = torch.empty(n, dtype=torch.float32, device=self.buf.device)
        self.kc_per_tile_row = n // (t1 - t0)
        return True

    # row views of the window (global row indices)
    def rows_view(self, t: torch.Tensor, r0: int, r1: int) -> torch.Tensor:
        b0 = self.lay.window[0]
        return t[r0 - b0:r1 - b0]

    def own(self, t: torch.Tensor) -> torch.Tensor:
        return self.rows_view(t, *self.lay.rows)

    def partial_rows(self, C: int, s0: int, s1: int) -> torch.Tensor:
        per = self.block_floats_c1 * C
        return self.partial[s0 * per:s1 * per]


class LocalComm:
    """N virtual ranks in one process (copies instead of messages)."""

    def shift_down(self, states, send, recv):
        """recv(state k) <- send(state k-1), k = 1..N-1."""
        for k in range(len(states) - 1, 0, -1):
            dst = recv(states[k])
            if dst is not None and dst.numel():
                dst.copy_(send(states[k - 1]))

    def shift_up(self, states, send, recv):
        """recv(state k) <- send(state k+1), k = 0..N-2."""
        for k in range(len(states) - 1):
            dst = recv(states[k])
            if dst is not None and dst.numel():
                dst.copy_(send(states[k + 1]))

    def start_shift(self, states, send, recv, direction):
        """shift_down (+1) / shift_up (-1) whose completion can be deferred:
        returns a finisher (here the copies are already done)."""
        (self.shift_down if direction > 0 else self.shift_up)(states, send, recv)
        return lambda: None

    def allreduce_max(self, states):
        m = torch.stack([s.mbits for s in states]).max(dim=0).values
        for s in states:
            s.mbits.copy_(m)

    def allreduce_sum(self, tensors):
        """In-place sum over the virtual ranks' tensors (rank order)."""
        tot = tensors[0].clone()
        for t in tensors[1:]:
            tot += t
        for t in tensors:
            t.copy_(tot)

    def shift(self, n, send, recv, direction):
        """recv(k) <- send(k - direction) for virtual ranks k (+1: down, -1: up)."""
        ks = range(n - 1, 0, -1) if direction > 0 else range(n - 1)
        for k in ks:
            dst = recv(k)
            if dst is not None and dst.numel():
                dst.copy_(send(k - direction))


class TorchComm:
    """Neighbour exchanges + max all-reduce over a torch.distributed group
    (NCCL for CUDA tensors; gloo works for the CPU tests of this logic)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def _peer(self, r):
        return self.dist.get_global_rank(self.group, r) if self.group is not None else r

    def _exchange(self, states, send, recv, direction):
        self.start_shift(states, send, recv, direction)()

    def start_shift(self, states, send, recv, direction):
        """Post this rank's half of a neighbour shift (NCCL runs it on its own
        stream once the current stream's prior work is done) and return a
        finisher that makes the current stream wait for it; work issued in
        between overlaps the transfer."""
        (st,) = states
        ops = []
        to = self.rank + direction
        frm = self.rank - direction
        if 0 <= to < self.size:
            t = send(st).contiguous()
            ops.append(self.dist.P2POp(self.dist.isend, t, self._peer(to), self.group))
        tmp, dst = None, None
        if 0 <= frm < self.size:
            dst = recv(st)
            tmp = dst if dst.is_contiguous() else torch.empty_like(dst)
            ops.append(self.dist.P2POp(self.dist.irecv, tmp, self._peer(frm), self.group))
        reqs = self.dist.batch_isend_irecv(ops) if ops else []

        def finish():
            for req in reqs:
                req.wait()
            if tmp is not None and tmp is not dst:
                dst.copy_(tmp)
        return finish

    def shift_down(self, states, send, recv):
        self._exchange(states, send, recv, +1)

    def shift_up(self, states, send, recv):
        self._exchange(states, send, recv, -1)

    def allreduce_max(self, states):
        (st,) = states
        self.dist.all_reduce(st.mbits, op=self.dist.ReduceOp.MAX, group=self.group)

    def allreduce_sum(self, tensors):
        (t,) = tensors
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)

    def shift(self, n, send, recv, direction):
        """This rank's half of recv(k) <- send(k - direction) (k = global rank)."""
        ops = []
        to, frm = self.rank + direction, self.rank - direction
        if 0 <= to < self.size:
            ops.append(self.dist.P2POp(self.dist.isend, send(self.rank).contiguous(),
                                       self._peer(to), self.group))
        tmp = None
        if 0 <= frm < self.size:
            dst = recv(self.rank)
            tmp = dst if dst.is_contiguous() else torch.empty_like(dst)
            ops.append(self.dist.P2POp(self.dist.irecv, tmp, self._peer(frm), self.group))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        if tmp is not None and tmp is not recv(self.rank):
            recv(self.rank).copy_(tmp)


class HostStagedComm(TorchComm):
    """TorchComm over a CPU backend (gloo) for device-resident strips: every
    message is staged through host memory (device -> host copy, gloo
    send/recv, host -> device copy).  Used to run the sharded algorithm in
    several processes where NCCL between them is not available (e.g. ranks
    sharing one GPU in a test); the exchanges complete before the call
    returns, so no rank's kernels ever wait on another's."""

    def start_shift(self, states, send, recv, direction):
        (st,) = states
        to = self.rank + direction
        frm = self.rank - direction
        ops, host_in, dst = [], None, None
        if 0 <= to < self.size:
            t = send(st).detach().to("cpu").contiguous()
            ops.append(self.dist.P2POp(self.dist.isend, t, self._peer(to), self.group))
        if 0 <= frm < self.size:
            dst = recv(st)
            host_in = torch.empty(tuple(dst.shape), dtype=dst.dtype)
            ops.append(self.dist.P2POp(self.dist.irecv, host_in, self._peer(frm), self.group))
        for req in (self.dist.batch_isend_irecv(ops) if ops else []):
            req.wait()
        if host_in is not None:
            dst.copy_(host_in)
        return lambda: None

    def allreduce_max(self, states):
        (st,) = states
        h = st.mbits.to("cpu")
        self.dist.all_reduce(h, op=self.dist.ReduceOp.MAX, group=self.group)
        st.mbits.copy_(h)

    def allreduce_sum(self, tensors):
        (t,) = tensors
        h = t.to("cpu")
        self.dist.all_reduce(h, op=self.dist.ReduceOp.SUM, group=self.group)
        t.copy_(h)

    def shift(self, n, send, recv, direction):
        ops = []
        to, frm = self.rank + direction, self.rank - direction
        if 0 <= to < self.size:
            ops.append(self.dist.P2POp(self.dist.isend, send(self.rank).detach().to("cpu")
                                       .contiguous(), self._peer(to), self.group))
        host_in = None
        if 0 <= frm < self.size:
            dst = recv(self.rank)
            host_in = torch.empty(tuple(dst.shape), dtype=dst.dtype)
            ops.append(self.dist.P2POp(self.dist.irecv, host_in, self._peer(frm), self.group))
        for req in (self.dist.batch_isend_irecv(ops) if ops else []):
            req.wait()
        if host_in is not None:
            recv(self.rank).copy_(host_in)


class ShardedDSG:
    """Adaptive DSG-NLM of a Hg x W image split in row strips.

    ``ranks`` lists the rank indices this process drives: ``[rank]`` with a
    TorchComm, or ``range(N)`` with a LocalComm (virtual shards)."""

    def __init__(self, params: PatchParams, Hg: int, W: int, nranks: int, ranks, comm,
                 device=None, kcache: bool = True):
        if params.pad_margin > min(Hg, W):
            raise ValueError(f"margin {params.pad_margin} exceeds min image extent {min(Hg, W)}")
        self.params = params
        self.comm = comm
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self.states = []
        for r in ranks:
            lay = StripLayout(Hg, W, params.window_radius, params.patch_side, nranks, r,
                              params.is_box)
            if lay.geom[3] == 2:
                raise ValueError("row-strip sharding needs the half-window sweep; this search "
                                 "radius / patch side only runs on one GPU")
            lay.validate()
            self.states.append(_RankState(lay, self.device))
            if kcache:
                self.states[-1].enable_kcache()
        self._taps = params._ctaps()

    # ---- host-side views ---------------------------------------------------
    def load(self, full_or_strips):
        """Fill each state's window from a full image (tensor/ndarray) — the
        data-loading path; ``denoise`` then exchanges halos itself."""
        for st in self.states:
            y0, y1 = st.lay.rows
            src = full_or_strips[y0:y1]
            st.own(st.buf).copy_(torch.as_tensor(src, dtype=torch.float32))

    def gather(self) -> torch.Tensor:
        return torch.cat([st.own(st.out) for st in self.states], dim=0)

    # ---- the sharded algorithm ----------------------------------------------
    def _sweep(self, st, pass_, C, x=None, tiles=None):
        """Strip sweep; ``x`` (a window-shaped buffer) replaces the guide as the
        filtered signal (frozen apply: pass 3 with the fixed guide).  ``tiles``
        = (ta, tb) restricts it to some of the strip's tile rows (same bits:
        tiles are independent)."""
        lay = st.lay
        b0, b1 = lay.window
        t0, t1 = lay.tile_rows
        ta, tb = (t0, t1) if tiles is None else tiles
        if tb <= ta:
            return
        part0, off, nslot = lay.part
        p = self.params
        kc = st.kcache
        if kc is not None and ta > t0:
            kc = kc[(ta - t0) * st.kc_per_tile_row:]
        L.call("pnp_dsg_strip_sweep", L.context(self.device.index), pass_, L.ptr(st.buf),
               L.ptr(st.buf if x is None else x), L.ptr(st.rs), lay.Hg, lay.W, b0, b1 - b0, ta,
               tb - ta, p.window_radius, p.patch_side, self._taps, float(p.bandwidth),
               L.ptr(st.partial), off + (ta - t0), nslot, L.ptr(kc))

    def _fixup(self, st, mode, inv_m=None, x=None, out=None, rows=None):
        lay = st.lay
        b0, b1 = lay.window
        y0, y1 = lay.rows if rows is None else rows
        if y1 <= y0:
            return
        part0, off, nslot = lay.part
        p = self.params
        L.call("pnp_dsg_strip_fixup", L.context(self.device.index), mode, L.ptr(st.partial),
               part0, nslot, lay.Hg, lay.W, p.window_radius, p.patch_side, int(lay.box), y0, y1,
               b0, b1 - b0,
               L.ptr(st.rs), L.ptr(st.kx), L.ptr(st.d), L.ptr(st.mbits), L.ptr(inv_m), L.ptr(x),
               L.ptr(out))

    @staticmethod
    def _split_rows(st):
        """Own rows that need the partial blocks received from the rank above
        (the first R rows) and the rest: ((y0, ya), (ya, y1))."""
        y0, y1 = st.lay.rows
        ya = min(y1, y0 + (st.lay.Rb if st.lay.rank > 0 else 0))
        return (y0, ya), (ya, y1)

    @staticmethod
    def _split_tiles(st):
        """Tile rows whose sweep reads the rs halo from the rank below (rows
        past y1 within rs_below rows of the tile) and the rest: (early, late)."""
        lay = st.lay
        t0, t1 = lay.tile_rows
        _, y1 = lay.rows
        if lay.rank == lay.nranks - 1:
            return (t0, t1), (t1, t1)
        tb = t0
        while tb < t1 and (tb + 1) * lay.TH + lay.rs_below <= y1:
            tb += 1
        return (t0, tb), (tb, t1)

    def _exchange_partials(self, C, start=False):
        def send(st):
            _, off, nslot = st.lay.part
            return st.partial_rows(C, nslot - st.lay.dti, nslot)

        def recv(st):
            _, off, _ = st.lay.part
            return st.partial_rows(C, 0, off)

        fin = self.comm.start_shift(self.states, send, recv, +1)
        if not start:
            fin()
        return fin

    def _exchange_rows(self, name, top=True, start=False):
        def up_send(st):   # our first rows -> rank above's bottom halo
            y0, y1 = st.lay.rows
            return st.rows_view(getattr(st, name), y0, y0 + st.lay.halo[1])

        def up_recv(st):
            y0, y1 = st.lay.rows
            b0, b1 = st.lay.window
            return st.rows_view(getattr(st, name), y1, b1)

        def down_send(st):  # our last rows -> rank below's top halo
            y0, y1 = st.lay.rows
            return st.rows_view(getattr(st, name), y1 - st.lay.halo[0], y1)

        def down_recv(st):
            y0, _ = st.lay.rows
            b0, _ = st.lay.window
            return st.rows_view(getattr(st, name), b0, y0)

        if not top and start:  # the bottom halo only, completion deferred
            return self.comm.start_shift(self.states, up_send, up_recv, -1)
        self.comm.shift_up(self.states, up_send, up_recv)
        if top and self.states[0].lay.halo[0] > 0:
            self.comm.shift_down(self.states, down_send, down_recv)
        return lambda: None

    def denoise(self) -> None:
        """One adaptive DSG-NLM of the loaded image; results in each state's out.
        Each neighbour exchange overlaps the work that does not need it: the
        partial blocks from the rank above only reach our first R rows (the
        other rows' fixups run while they travel), the rs halo from the rank
        below only feeds our last tile row(s) (the others' sweeps run first)."""
        self._exchange_rows("buf")
        for st in self.states:
            self._sweep(st, 0, 1)
        fin = self._exchange_partials(1, start=True)
        for st in self.states:
            self._fixup(st, 0, rows=self._split_rows(st)[1])
        fin()
        for st in self.states:
            self._fixup(st, 0, rows=self._split_rows(st)[0])
        fin = self._exchange_rows("rs", top=False, start=True)  # y channels read rows below
        for st in self.states:
            self._sweep(st, 1, 2, tiles=self._split_tiles(st)[0])
        fin()
        for st in self.states:
            self._sweep(st, 1, 2, tiles=self._split_tiles(st)[1])
        fin = self._exchange_partials(2, start=True)
        for st in self.states:
            st.mbits.zero_()
            self._fixup(st, 1, rows=self._split_rows(st)[1])
        fin()
        for st in self.states:
            self._fixup(st, 1, rows=self._split_rows(st)[0])
        self.comm.allreduce_max(self.states)
        for st in self.states:
            lay = st.lay
            b0, b1 = lay.window
            y0, y1 = lay.rows
            L.call("pnp_dsg_strip_finalize", L.context(self.device.index), L.ptr(st.kx),
                   L.ptr(st.d), L.ptr(st.buf), L.ptr(st.out), L.ptr(st.mbits), lay.Hg, lay.W,
                   y0, y1, b0, b1 - b0)

    def alpha(self) -> float:
        return float(self.states[0].mbits.view(torch.float32)[0])


def sharded_dsg_nlm_denoise(image: torch.Tensor, params: PatchParams, nshards: int,
                            kcache: bool = True) -> torch.Tensor:
    """Virtual-shard run on one device (N strips, LocalComm): same bits as
    ``dsg_nlm_denoise(image, params)``; exercises the multi-GPU algorithm."""
    H, W = image.shape
    sh = ShardedDSG(params, H, W, nshards, range(nshards), LocalComm(), device=image.device,
                    kcache=kcache)
    sh.load(image)
    sh.denoise()
    return sh.gather()


# ---------------------------------------------------------------------------
# Sharded linearized PnP-ADMM for super-resolution
# ---------------------------------------------------------------------------

class ShardedSRADMM:
    """Linearized PnP-ADMM (solver.py:199-235) on one large SR image split in
    row strips, with a frozen-guide DSG denoiser.  Per rank and iteration:

        x halo (blur radius rows)                      [P2P]
        r = A x - y on own low-res rows (+ 0.5||r||^2) [strip residual]
        r halo (ceil(radius/factor) low-res rows)      [P2P]
        grad = A^T r on own rows, x-update             [strip adjoint]
        z halo (rows the DSG sweep reads below)        [P2P]
        v = W z: strip sweep over the frozen guide's k cache / filter, partial
        blocks -> next rank, fixup with the global 1/m [P2P]
        u-update + primal / dual / PSNR partial sums   [all-reduce]

    Strip boundaries are DSG tile rows (multiples of TH, pnp_dsg_geometry; the
    decimation factor must divide), every operator reads global rows through
    halos, so x, z, v, u are bit-identical to the single-GPU solver; the
    records' float64 sums differ only in summation order.  ``ranks`` /
    ``comm`` as in ShardedDSG (LocalComm = virtual ranks on one device)."""

    def __init__(self, op, params: PatchParams, Hg: int, W: int, nranks: int, ranks, comm,
                 device=None, kcache: bool = True):
        self.op, self.params, self.comm = op, params, comm
        self.Hg, self.W, self.k = Hg, W, op.factor
        self.rad = op.radius
        self.dsg = ShardedDSG(params, Hg, W, nranks, ranks, comm, device=device, kcache=kcache)
        self.device = self.dsg.device
        TH = self.dsg.states[0].lay.TH
        if Hg % self.k or W % self.k or TH % self.k:
            raise ValueError(f"factor {self.k} must divide the image and the strip tile height {TH}")
        self.hr = -(-self.rad // self.k)
        self.ranks = list(ranks)
        self.nranks = nranks
        self.st = {}
        d = self.device
        for rk, ds in zip(self.ranks, self.dsg.states):
            y0, y1 = ds.lay.rows
            if (y1 - y0 < max(self.rad, ds.lay.halo[1]) or (y1 - y0) // self.k < self.hr):
                raise ValueError("strip too thin for the blur / DSG halos")
            e = {"ds": ds, "rows": (y0, y1)}
            e["xr"] = (max(0, y0 - self.rad), min(Hg, y1 + self.rad))
            e["rr"] = (max(0, y0 // self.k - self.hr), min(Hg // self.k, y1 // self.k + self.hr))
            e["x"] = torch.zeros((e["xr"][1] - e["xr"][0], W), dtype=torch.float32, device=d)
            e["r"] = torch.zeros((e["rr"][1] - e["rr"][0], W // self.k), dtype=torch.float32,
                                 device=d)
            e["y"] = torch.zeros(((y1 - y0) // self.k, W // self.k), dtype=torch.float32, device=d)
            own = (y1 - y0, W)
            e["u"] = torch.zeros(own, dtype=torch.float32, device=d)
            e["grad"] = torch.zeros(own, dtype=torch.float32, device=d)
            e["gt"] = None
            e["z"] = torch.zeros_like(ds.buf)   # DSG window (halos the sweep reads)
            e["v"] = torch.zeros_like(ds.buf)   # window-shaped: the apply fixup writes own rows
            e["flags"] = None
            self.st[rk] = e
        self._taps = op._taps
        self.inv_m = torch.zeros(1, dtype=torch.float32, device=d)

    # ---- helpers ----------------------------------------------------------
    @staticmethod
    def _own(e, name):
        t = e[name]
        if name in ("x",):
            a = e["xr"][0]
        elif name in ("z", "v", "v_prev"):
            a = e["ds"].lay.window[0]
        else:
            return t
        y0, y1 = e["rows"]
        return t[y0 - a:y1 - a]

    def _halo(self, name, r0_key, top, bottom, lowres=False):
        """Fill ``name``'s halo rows (``top`` above, ``bottom`` below own rows)
        from the neighbouring ranks' own edge rows."""
        k = self.k if lowres else 1

        def edges(rk):
            e = self.st[rk]
            y0, y1 = e["rows"]
            base = e[r0_key][0] if r0_key else e["ds"].lay.window[0]
            return e[name], y0 // k - base, y1 // k - base

        def bottom_recv(rk):
            t, a, b = edges(rk)
            return t[b:b + bottom]

        def bottom_send(rk):
            t, a, b = edges(rk)
            return t[a:a + bottom]

        def top_recv(rk):
            t, a, b = edges(rk)
            return t[a - top:a]

        def top_send(rk):
            t, a, b = edges(rk)
            return t[b - top:b]

        if bottom:
            self.comm.shift(self.nranks, bottom_send, bottom_recv, -1)
        if top:
            self.comm.shift(self.nranks, top_send, top_recv, +1)

    # ---- loading -------------------------------------------------------------
    def load(self, y_full, guide_full, truth_full=None, x0_full=None):
        """Distribute the observation (low-res), the guide and optionally the
        ground truth / start point (full-size host or device arrays)."""
        self.dsg.load(guide_full)
        for e in self.st.values():
            y0, y1 = e["rows"]
            e["y"].copy_(torch.as_tensor(y_full[y0 // self.k:y1 // self.k], dtype=torch.float32))
            if truth_full is not None:
                e["gt"] = torch.as_tensor(truth_full[y0:y1], dtype=torch.float32).to(
                    self.device).contiguous()
            if x0_full is not None:
                self._own(e, "x").copy_(torch.as_tensor(x0_full[y0:y1], dtype=torch.float32))
        if x0_full is None:  # make_sr_problem's start: k^2 A^T y (solver.py:340)
            self._exchange_lr("y_as_r")
            for e in self.st.values():
                y0, y1 = e["rows"]
                self._adjoint(e, e["r"], self._own(e, "x"))
                self._own(e, "x").mul_(float(self.k * self.k))

    def _exchange_lr(self, what):
        for e in self.st.values():
            a = e["rr"][0]
            y0, y1 = e["rows"]
            src = e["y"] if what == "y_as_r" else None
            e["r"][y0 // self.k - a:y1 // self.k - a].copy_(src)
        self._halo("r", "rr", self.hr, self.hr, lowres=True)

    def _adjoint(self, e, rbuf, out):
        y0, y1 = e["rows"]
        a, b = e["rr"]
        o = self.op
        L.call("pnp_sr_strip_adjoint", L.context(self.device.index), L.ptr(rbuf), L.ptr(out),
               self.Hg, self.W, a, b - a, y0, y1 - y0, self._taps, o.radius, o.factor, o._bnd)

    # ---- the sharded guide freeze -------------------------------------------
    def freeze(self):
        """FrozenGuide.__init__ (denoise.py:367-373) on the strips: mass sweep,
        rs, row sums d, global max m -> 1/m (bit-identical to one GPU)."""
        dsg = self.dsg
        dsg._exchange_rows("buf")
        for st in dsg.states:
            dsg._sweep(st, 0, 1)
        dsg._exchange_partials(1)
        for st in dsg.states:
            dsg._fixup(st, 0)
        dsg._exchange_rows("rs", top=False)
        for st in dsg.states:
            dsg._sweep(st, 2, 1)
        dsg._exchange_partials(1)
        for st in dsg.states:
            st.mbits.zero_()
            dsg._fixup(st, 2)
        self.comm.allreduce_max(dsg.states)
        m = dsg.states[0].mbits.view(torch.float32)
        self.inv_m.copy_(1.0 / m)  # IEEE reciprocal, the single-GPU 1/m
        return float(m[0])

    # ---- the solver ----------------------------------------------------------
    def run(self, config):
        """config: SolverConfig (rho, alpha, max_iters, constraint).  Returns
        the per-iteration records (index, primal, dual, psnr, objective)."""
        from .image import bounds
        lo, hi = bounds(config.constraint)
        rho, alpha = float(config.rho), float(config.alpha)
        mu = 1.0 / (alpha + rho)
        n_total = self.Hg * self.W
        iters = config.max_iters
        ctx = L.context(self.device.index)
        o = self.op
        for e in self.st.values():
            xo = self._own(e, "x")
            L.call("pnp_project", ctx, L.ptr(xo), L.ptr(xo), xo.numel(), lo, hi)
            self._own(e, "v").copy_(xo)
            e["u"].zero_()
            e["stats"] = torch.zeros((iters, 1, 4), dtype=torch.float64, device=self.device)
            e["obj"] = torch.zeros((iters + 1, 1), dtype=torch.float64, device=self.device)
            e["flags"] = torch.zeros(iters, dtype=torch.int32, device=self.device)
        for k in range(1, iters + 1):
            self._halo("x", "xr", self.rad, self.rad)
            for e in self.st.values():
                y0, y1 = e["rows"]
                a, b = e["xr"]
                ra = e["rr"][0]
                r_own = e["r"][y0 // self.k - ra:y1 // self.k - ra]
                L.call("pnp_sr_strip_residual", ctx, L.ptr(e["x"]), L.ptr(e["y"]), L.ptr(r_own),
                       self.Hg, self.W, a, b - a, y0 // self.k, (y1 - y0) // self.k, self._taps,
                       o.radius, o.factor, o._bnd, L.ptr(e["obj"][k - 1]))
            self._halo("r", "rr", self.hr, self.hr, lowres=True)
            for e in self.st.values():
                self._adjoint(e, e["r"], e["grad"])
                xo, zo, vo = self._own(e, "x"), self._own(e, "z"), self._own(e, "v")
                L.call("pnp_admm_xupdate", ctx, L.ptr(xo), L.ptr(vo), L.ptr(e["u"]),
                       L.ptr(e["grad"]), L.ptr(zo), xo.numel(), mu, alpha, rho, lo, hi,
                       L.ptr(e["flags"][k - 1:k]))
            self._halo("z", None, 0, self.dsg.states[0].lay.halo[1])
            for e in self.st.values():
                e["v_prev"] = e["v"]
                e["v"] = torch.zeros_like(e["z"])
                self.dsg._sweep(e["ds"], 3, 1, x=e["z"])
            self.dsg._exchange_partials(1)
            for e in self.st.values():
                self.dsg._fixup(e["ds"], 3, inv_m=self.inv_m, x=e["z"], out=e["v"])
                xo, vo, vp = self._own(e, "x"), self._own(e, "v"), self._own(e, "v_prev")
                L.call("pnp_admm_uupdate", ctx, L.ptr(e["u"]), L.ptr(xo), L.ptr(vo), L.ptr(vp),
                       L.ptr(e["gt"]), 1, xo.numel(), rho, L.ptr(e["stats"][k - 1]),
                       L.ptr(e["flags"][k - 1:k]))
        # objective of the final iterate
        self._halo("x", "xr", self.rad, self.rad)
        for e in self.st.values():
            y0, y1 = e["rows"]
            a, b = e["xr"]
            ra = e["rr"][0]
            L.call("pnp_sr_strip_residual", ctx, L.ptr(e["x"]), L.ptr(e["y"]),
                   L.ptr(e["r"][y0 // self.k - ra:y1 // self.k - ra]), self.Hg, self.W, a, b - a,
                   y0 // self.k, (y1 - y0) // self.k, self._taps, o.radius, o.factor, o._bnd,
                   L.ptr(e["obj"][iters]))
        es = list(self.st.values())
        self.comm.allreduce_sum([e["stats"] for e in es])
        self.comm.allreduce_sum([e["obj"] for e in es])
        self.comm.allreduce_sum([e["flags"] for e in es])
        st = es[0]["stats"].cpu().numpy()
        ob = es[0]["obj"].cpu().numpy()
        fl = es[0]["flags"].cpu().numpy()
        bad = [i for i in range(iters) if fl[i]]
        if bad:
            from .solver import DivergenceError
            raise DivergenceError(f"non-finite iterate at iteration {bad[0] + 1}")
        import math
        recs = []
        for i in range(iters):
            mse = st[i, 0, 2] / n_total
            q = math.inf if mse == 0 else 10.0 * math.log10(1.0 / mse)
            recs.append((i + 1, st[i, 0, 0] / n_total, st[i, 0, 1] / n_total,
                         q if es[0]["gt"] is not None else math.nan, ob[i + 1, 0]))
        return recs

    def gather(self) -> torch.Tensor:
        """v of every local rank, concatenated (the full image for LocalComm)."""
        return torch.cat([self._own(self.st[rk], "v") for rk in self.ranks], dim=0)


def sharded_linearized_pnp_admm_sr(op, y, guide, params: PatchParams, config, nshards: int,
                                   ground_truth=None, kcache: bool = True):
    """Virtual-shard run on one device (N strips, LocalComm) of the frozen-guide
    SR ADMM; same v as ``linearized_pnp_admm`` with ``freeze_guide(guide)``."""
    H, W = guide.shape
    sh = ShardedSRADMM(op, params, H, W, nshards, range(nshards), LocalComm(), kcache=kcache)
    sh.load(y, guide, ground_truth)
    sh.freeze()
    recs = sh.run(config)
    return sh.gather(), recs
