"""Slab decomposition of the fused 3-D pseudo-time solve over P GPUs.

SURVEY §8(e): one process per GPU; the grid is split along axis 0 (the
memory-slowest axis, periodic in BASELINE configs 4 and 5) into contiguous
slabs of ``nl = n0 / P`` planes, each stored with ``G`` ghost planes per side.
One pseudo-step:

* before each RK stage, exchange the stage input's ghost planes with both
  ring neighbours (``send/recv``, NCCL over NVLink);
* run the fused stage kernel on the slab interior (``wd_dist_stage``);
* filter axis 0 on full x-lines.  Exact arithmetic: pack the slab into P
  chunks, ``all_to_all`` to pencils ``(n0, n1/P, n2)``, sweep, ``all_to_all``
  back (bit-identical to one GPU).  Fast arithmetic (default there): the
  partitioned solve of ``csrc/wd_dist_filter0.cuh`` -- ghost exchange of the
  filter input, then per line one forward carry and one backward carry
  ``all_gather``-ed between three local kernels (2 + 1 doubles per line per
  rank instead of two transposes of the whole slab: ~6 MB vs ~234 MB per GPU
  and step at 512^3, P = 8);
* filter axes 1 and 2 on the slab; the last sweep accumulates the local
  ``max|Δφ|``, ``max|φ|`` and non-finite flag;
* ``all_reduce(max)`` of those three words, then the stop test.

With the transposed axis-0 filter every node and every filter line sees
exactly the operations of the single-GPU path, so the decomposed solve is
bit-identical to it; the partitioned filter solves the same linear system
with another association (round-off level; checked by
``tests/test_gpu_dist.py`` with P simulated ranks on one GPU).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat

GHOST = 7  # >= 4 + R (exact axis-0 windows) and >= 2R (fast mode), R <= 3


@dataclass(frozen=True)
class Slab:
    """Rank ``rank``'s share of axis 0: global planes [lo, lo + nl)."""

    n0: int
    P: int
    rank: int
    G: int = GHOST

    @property
    def nl(self) -> int:
        return self.n0 // self.P

    @property
    def lo(self) -> int:
        return self.rank * self.nl

    @property
    def left(self) -> int:
        return (self.rank - 1) % self.P

    @property
    def right(self) -> int:
        return (self.rank + 1) % self.P

    def check(self, n1: int):
        if self.n0 % self.P:
            raise ValueError(f"axis 0 ({self.n0}) must divide evenly over {self.P} ranks")
        if n1 % self.P:
            raise ValueError(f"axis 1 ({n1}) must divide evenly over {self.P} ranks")
        if self.nl < self.G:
            raise ValueError(f"slab of {self.nl} planes is thinner than {self.G} ghost planes")


def split_global(field, P):
    """Global (n0, n1, n2) array -> list of P ghosted slabs (ghosts zero)."""
    n0 = field.shape[0]
    out = []
    for r in range(P):
        s = Slab(n0, P, r)
        g = np.zeros((s.nl + 2 * s.G,) + field.shape[1:])
        g[s.G:s.G + s.nl] = field[s.lo:s.lo + s.nl]
        out.append(g)
    return out


# ------------------------------------------------------------- communicators
class TorchComm:
    """One rank of a torch.distributed group (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def halo(self, slabs, slab: Slab):
        """Fill the ghost planes of this rank's (nl + 2G, ...) tensor."""
        self.halo_finish(self.halo_start(slabs, slab), slabs, slab)

    def halo_start(self, slabs, slab: Slab):
        """Post the ghost-plane exchange; the caller may enqueue work that
        does not read the ghost planes before halo_finish."""
        (t,) = slabs
        G, nl = slab.G, slab.nl
        if self.P == 1:
            t[:G].copy_(t[nl:nl + G])
            t[nl + G:].copy_(t[G:2 * G])
            return None
        d = self.dist
        lo = t.new_empty(t[:G].shape)
        hi = t.new_empty(t[:G].shape)
        # posting order matters when left == right (P = 2): point-to-point
        # ops between one pair of ranks match in the order they are posted
        ops = [d.P2POp(d.isend, t[nl:nl + G].contiguous(), slab.right, self.group),
               d.P2POp(d.irecv, lo, slab.left, self.group),
               d.P2POp(d.isend, t[G:2 * G].contiguous(), slab.left, self.group),
               d.P2POp(d.irecv, hi, slab.right, self.group)]
        return d.batch_isend_irecv(ops), lo, hi

    def halo_finish(self, handle, slabs, slab: Slab):
        if handle is None:
            return
        (t,) = slabs
        reqs, lo, hi = handle
        for req in reqs:
            req.wait()
        t[:slab.G].copy_(lo)
        t[slab.nl + slab.G:].copy_(hi)

    def alltoall(self, outs, ins):
        (o,), (i,) = outs, ins
        if self.P == 1:
            o.copy_(i)
            return
        self.dist.all_to_all_single(o, i, group=self.group)

    def allgather(self, outs, ins):
        """outs[0] (P * len(ins[0]),) <- every rank's ins[0], rank order."""
        (o,), (i,) = outs, ins
        if self.P == 1:
            o.copy_(i)
            return
        self.dist.all_gather_into_tensor(o, i, group=self.group)

    def allreduce_max(self, ts):
        (t,) = ts
        if self.P > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)


class LocalComm:
    """P logical ranks in one process (device copies stand in for NVLink).
    Used to check the decomposition on one GPU: no kernel ever waits on
    another rank's kernel."""

    def __init__(self, P):
        self.P = P

    def halo_start(self, slabs, slab: Slab):
        self.halo(slabs, slab)
        return None

    def halo_finish(self, handle, slabs, slab: Slab):
        return None

    def halo(self, slabs, slab: Slab):
        G, nl = slab.G, slab.nl
        P = self.P
        lows = [t[G:2 * G].clone() for t in slabs]
        highs = [t[nl:nl + G].clone() for t in slabs]
        for r, t in enumerate(slabs):
            t[:G].copy_(highs[(r - 1) % P])
            t[nl + G:].copy_(lows[(r + 1) % P])

    def alltoall(self, outs, ins):
        P = self.P
        chunks = [i.view(P, -1) for i in ins]
        for r, o in enumerate(outs):
            ov = o.view(P, -1)
            for s in range(P):
                ov[s].copy_(chunks[s][r])

    def allgather(self, outs, ins):
        P = self.P
        for o in outs:
            ov = o.view(P, -1)
            for s_ in range(P):
                ov[s_].copy_(ins[s_])

    def allreduce_max(self, ts):
        import torch
        m = torch.stack(list(ts)).max(dim=0).values
        for t in ts:
            t.copy_(m)


# ------------------------------------------------------------------ solver
class DistributedSolve:
    """Fused 3-D pseudo-time solve on the slabs of ``ranks`` (one entry per
    local logical rank: 1 under torchrun, P in the simulated mode)."""

    def __init__(self, dims, spacing, faces, scheme, formulation, filter_config, cfl, tol,
                 max_iters, arith, comm, ranks, ref_length=1.0, filter0=None, overlap=True):
        import torch
        from ._context import NativeSolver
        from .grid import CurvilinearGrid
        self.torch = torch
        self.comm = comm
        n0, n1, n2 = dims
        P = comm.P
        if faces.get("imin") != "periodic":
            raise ValueError("slab decomposition needs a periodic axis 0")
        if filter_config is None:
            raise ValueError("the distributed path runs the filtered scheme")
        self.dims = dims
        self.slabs = [Slab(n0, P, r) for r in ranks]
        for s in self.slabs:
            s.check(n1)
        s0 = self.slabs[0]
        self.nl, self.G = s0.nl, s0.G
        gdims = (self.nl + 2 * self.G, n1, n2)
        # local geometry: ghosted slab, axis 0 open (ghosts carry the wrap)
        lfaces = {k: v for k, v in faces.items() if k not in ("imin", "imax")}
        per = (False, faces.get("jmin") == "periodic", faces.get("kmin") == "periodic")
        self.per = per
        g = CurvilinearGrid._analytic((0.0, 0.0, 0.0), spacing, gdims, ref_length, per,
                                      [spacing[d] * gdims[d] for d in range(3)])
        self.ctxs = []
        self.hists = []
        for _ in ranks:
            ctx = NativeSolver(g, lfaces, None, scheme, formulation, filter_config, cfl, tol,
                               max_iters, arith=arith)
            if not ctx.fused:
                raise ValueError("configuration is not on the fused 3-D path")
            nat.check(ctx.lib.wd_dist_configure(ctx.ptr, self.G, self.G + self.nl))
            self.ctxs.append(ctx)
        self.lib = self.ctxs[0].lib
        f64 = dict(dtype=torch.float64, device="cuda")
        R = len(ranks)
        self.A = [torch.zeros(gdims, **f64) for _ in range(R)]
        self.B = [torch.zeros(gdims, **f64) for _ in range(R)]
        self.Pa = [torch.zeros(gdims, **f64) for _ in range(R)]
        self.Pb = [torch.zeros(gdims, **f64) for _ in range(R)]
        nlc = self.nl * n1 * n2
        self.send = [torch.empty(nlc, **f64) for _ in range(R)]
        self.pen = [torch.empty(nlc, **f64) for _ in range(R)]
        self.pen2 = [torch.empty(nlc, **f64) for _ in range(R)]
        self.back = [torch.empty(nlc, **f64) for _ in range(R)]
        self.slab1 = [torch.empty((self.nl, n1, n2), **f64) for _ in range(R)]
        self.slab2 = [torch.empty((self.nl, n1, n2), **f64) for _ in range(R)]
        self.stats = [torch.zeros(3, dtype=torch.int64, device="cuda") for _ in range(R)]
        # stage kernels on the planes that need no ghost while the ghost
        # planes are in flight, then the 2 x G boundary planes
        self.overlap = bool(overlap) and self.nl >= 2 * self.G + 8
        # axis-0 filter: "partitioned" (fast arithmetic) or "transpose"
        self.filter0 = filter0 or ("partitioned" if arith == "fast" else "transpose")
        if self.filter0 not in ("partitioned", "transpose"):
            raise ValueError(f"unknown axis-0 filter mode {self.filter0!r}")
        if self.filter0 == "partitioned" and arith != "fast":
            raise ValueError("the partitioned axis-0 filter is a fast-arithmetic path")
        lines = n1 * n2
        self.mineA = [torch.empty(2 * lines, **f64) for _ in range(R)]
        self.mineB = [torch.empty(lines, **f64) for _ in range(R)]
        self.gathA = [torch.empty(P * 2 * lines, **f64) for _ in range(R)]
        self.gathB = [torch.empty(P * lines, **f64) for _ in range(R)]
        for ctx in self.ctxs:
            h = torch.zeros(max(max_iters, 1), **f64)
            self.hists.append(h)
        self._bound = False

    # -- state
    def set_state(self, local_slabs):
        """local_slabs: per local rank, (nl, n1, n2) arrays (numpy or torch)."""
        torch = self.torch
        for A, s in zip(self.A, local_slabs):
            t = s if isinstance(s, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(s))
            A[self.G:self.G + self.nl].copy_(t.to(A.device))
        for ctx, A, h in zip(self.ctxs, self.A, self.hists):
            # wd_bind applies the (wall) BCs of the local geometry and resets status
            nat.check(self.lib.wd_bind(ctx.ptr, A.data_ptr(), h.data_ptr()))
        self._bound = True

    def state(self):
        return [A[self.G:self.G + self.nl] for A in self.A]

    def _interior(self, t):
        return t[self.G:self.G + self.nl]

    def step(self):
        torch = self.torch
        if isinstance(self.comm, LocalComm):
            self._step()
            return
        # one rank per process: run torch-side transfers on the solver stream
        with torch.cuda.stream(self.ctxs[0].stream()):
            self._step()

    def _step(self):
        lib, comm = self.lib, self.comm
        n0, n1, n2 = self.dims
        P, nl = comm.P, self.nl
        m1 = n1 // P
        R = len(self.ctxs)
        bufs = [self.A, self.Pa, self.Pb, self.Pa]
        outs = [self.Pa, self.Pb, self.Pa, self.Pb]
        G = self.G
        for s in range(4):
            self._sync()
            h = comm.halo_start(bufs[s], self.slabs[0])

            def launch(lo, hi):
                for r in range(R):
                    nat.check(lib.wd_dist_configure(self.ctxs[r].ptr, lo, hi))
                    nat.check(lib.wd_dist_stage(self.ctxs[r].ptr, s + 1, self.A[r].data_ptr(),
                                                bufs[s][r].data_ptr(), outs[s][r].data_ptr()))
            if self.overlap:
                # planes [2G, nl): every stencil reach (<= G planes) stays
                # inside the rank's own planes
                launch(2 * G, nl)
                comm.halo_finish(h, bufs[s], self.slabs[0])
                self._sync()
                launch(G, 2 * G)
                launch(nl, nl + G)
            else:
                comm.halo_finish(h, bufs[s], self.slabs[0])
                self._sync()
                launch(G, G + nl)
        for r in range(R):
            nat.check(lib.wd_dist_configure(self.ctxs[r].ptr, G, G + nl))
        streams = [self.ctxs[r].lib.wd_get_stream(self.ctxs[r].ptr) for r in range(R)]
        if self.filter0 == "partitioned":
            self._filter0_partitioned()
        else:
            self._filter0_transpose(streams)
        for r in range(R):
            nat.check(lib.wd_dist_filter(self.ctxs[r].ptr, 1, self.slab1[r].data_ptr(),
                                         self.slab2[r].data_ptr(), nl, n1, n2,
                                         int(self.per[1]), None))
            nat.check(lib.wd_dist_filter(self.ctxs[r].ptr, 2, self.slab2[r].data_ptr(),
                                         self._interior(self.B[r]).data_ptr(), nl, n1, n2,
                                         int(self.per[2]), self._interior(self.A[r]).data_ptr()))
            nat.check(lib.wd_dist_stats(self.ctxs[r].ptr, self.stats[r].data_ptr()))
        self._sync()
        comm.allreduce_max(self.stats)
        self._sync()
        for r in range(R):
            nat.check(lib.wd_dist_finalize(self.ctxs[r].ptr, self.stats[r].data_ptr()))
        self.A, self.B = self.B, self.A

    def _filter0_partitioned(self):
        """Axis-0 filter of the stage-4 output Pb -> slab1, rows split over
        the ranks (wd_dist_filter0: three local phases, two all_gathers)."""
        lib, comm = self.lib, self.comm
        n0, n1, n2 = self.dims
        P = comm.P
        R = len(self.ctxs)
        self._sync()
        comm.halo(self.Pb, self.slabs[0])
        self._sync()

        def phase(ph, mine):
            for r in range(R):
                nat.check(lib.wd_dist_filter0(
                    self.ctxs[r].ptr, ph, self.Pb[r].data_ptr(), self.slab1[r].data_ptr(), n0,
                    n1, n2, self.G, P, self.slabs[r].rank, self.gathA[r].data_ptr(),
                    self.gathB[r].data_ptr(), mine[r].data_ptr()))
        phase(1, self.mineA)
        self._sync()
        comm.allgather(self.gathA, self.mineA)
        self._sync()
        phase(2, self.mineB)
        self._sync()
        comm.allgather(self.gathB, self.mineB)
        self._sync()
        phase(3, self.mineB)

    def _filter0_transpose(self, streams):
        """Axis-0 filter on pencils (n0, n1/P, n2): pack, all_to_all, sweep,
        all_to_all back, unpack -> slab1 (bit-identical to one GPU)."""
        lib, comm = self.lib, self.comm
        n0, n1, n2 = self.dims
        P, nl = comm.P, self.nl
        m1 = n1 // P
        R = len(self.ctxs)
        for r in range(R):
            x = self._interior(self.Pb[r])
            nat.check(lib.wd_dist_pack(x.data_ptr(), self.send[r].data_ptr(), nl, n1, n2, P,
                                       streams[r]))
        self._sync()
        comm.alltoall(self.pen, self.send)
        self._sync()
        for r in range(R):
            nat.check(lib.wd_dist_filter(self.ctxs[r].ptr, 0, self.pen[r].data_ptr(),
                                         self.pen2[r].data_ptr(), n0, m1, n2, 1, None))
        self._sync()
        comm.alltoall(self.back, self.pen2)
        self._sync()
        for r in range(R):
            nat.check(lib.wd_dist_unpack(self.back[r].data_ptr(), self.slab1[r].data_ptr(), nl,
                                         n1, n2, P, streams[r]))

    def _sync(self):
        """Simulated ranks use one stream per logical rank: order them
        around the device-copy transfers.  With one rank per process all work
        shares the solver stream and needs no host synchronisation."""
        if isinstance(self.comm, LocalComm):
            self.torch.cuda.synchronize()

    def status(self, r=0):
        st = nat.Status()
        nat.check(self.lib.wd_read_status(self.ctxs[r].ptr, ctypes.byref(st)))
        return st

    def history(self, r=0):
        st = self.status(r)
        return self.hists[r][:st.iters].cpu().numpy()

    def close(self):
        for c in self.ctxs:
            c.close()
