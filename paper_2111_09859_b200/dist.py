"""Slab decomposition of the pseudo-time solve over P GPUs.

One process per GPU; rank r owns the planes ``[r n0/P, (r+1) n0/P)`` of the
periodic axis 0 (the memory-slowest axis: ghost planes and slabs are
contiguous).  The whole step program lives in the native library
(``csrc/wd_dist.cuh``, C ABI ``wd_comm_*`` / ``wd_dist_*``):

* fused 3-D path (BASELINE config 4): ghost-plane exchange per RK stage,
  overlapped with the interior planes; axis-0 filter as a partitioned solve
  (fast arithmetic: one local scan kernel, ONE all_gather of three doubles
  per line, one fix-up) or a slab <-> pencil transpose pair (exact arithmetic:
  bit-identical to one GPU); one ``all_reduce(max)`` of three words per step;
* generic path (compact / curvilinear / LAD / curvature / Poisson / UW,
  BASELINE config 5): every operator ALONG axis 0 runs on pencils between
  two all_to_all transposes, everything else is local -- bit-identical.

Communicators:

* :class:`NcclComm` -- the product path: NCCL inside the library
  (``wd_comm_init``), the k-step CUDA graph contains the collectives;
* :class:`TorchComm` -- the same program over any ``torch.distributed``
  backend through host callbacks (gloo stages through the host; used by the
  multi-process tests on one GPU or none);
* :class:`LocalComm` -- P logical ranks in one process, one thread each
  (device copies stand in for NVLink; every wait is a host barrier, so no
  kernel ever waits on another rank's kernel).

``solve_steady(grid, boundary, config, comm=...)`` is the user entry point.
"""
from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np

from . import _native as nat

GHOST = 7  # fused path: >= 4 + R (exact axis-0 windows) and >= 2R (fast), R <= 3


@dataclass(frozen=True)
class Slab:
    """Rank ``rank``'s share of axis 0: global planes [lo, lo + nl)."""

    n0: int
    P: int
    rank: int

    @property
    def nl(self) -> int:
        return self.n0 // self.P

    @property
    def lo(self) -> int:
        return self.rank * self.nl

    @property
    def hi(self) -> int:
        return self.lo + self.nl

    @property
    def left(self) -> int:
        return (self.rank - 1) % self.P

    @property
    def right(self) -> int:
        return (self.rank + 1) % self.P

    def check(self):
        if self.n0 % self.P:
            raise ValueError(f"axis 0 ({self.n0}) must divide evenly over {self.P} ranks")


def split_global(field, P):
    """Global (n0, ...) array -> list of P contiguous slabs."""
    n0 = field.shape[0]
    if n0 % P:
        raise ValueError(f"axis 0 ({n0}) must divide evenly over {P} ranks")
    nl = n0 // P
    return [np.ascontiguousarray(field[r * nl:(r + 1) * nl]) for r in range(P)]


class _DevArray:
    """Raw device memory as a ``__cuda_array_interface__`` object."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 2}


def dev_view(ptr, n, dtype="f8"):
    """Zero-copy torch view of ``n`` elements of device memory at ``ptr``."""
    import torch
    return torch.as_tensor(_DevArray(ptr, n, "<" + dtype), device="cuda")


# ------------------------------------------------------------- communicators
class _Comm:
    """Owner of a native ``wd_comm``."""

    ptr = None
    P = 1
    rank = 0

    def close(self):
        if getattr(self, "ptr", None) is not None and self.ptr.value:
            nat.lib().wd_comm_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # collectives used outside the step program (collecting a result)
    def allgather(self, mine, stream=None):
        """(P * n,) tensor of every rank's ``mine`` (n,), rank order."""
        import torch
        out = torch.empty(self.P * mine.numel(), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        nat.check(nat.lib().wd_comm_allgather(self.ptr, mine.data_ptr(), out.data_ptr(),
                                              mine.numel(), stream))
        torch.cuda.synchronize()
        return out


class NcclComm(_Comm):
    """NCCL communicator owned by the library (``wd_comm_init``).  ``nccl_id``
    is the 128-byte id made by rank 0 (:meth:`unique_id`); :meth:`from_torch`
    broadcasts it over an initialised ``torch.distributed`` group."""

    def __init__(self, rank: int, nranks: int, nccl_id: bytes | None = None):
        lib = nat.lib()
        self.rank, self.P = int(rank), int(nranks)
        if self.P > 1 and (nccl_id is None or len(nccl_id) != 128):
            raise ValueError("a 128-byte NCCL unique id is required for more than one rank")
        buf = ctypes.create_string_buffer(nccl_id or b"", 128)
        ptr = ctypes.c_void_p()
        nat.check(lib.wd_comm_init(buf, self.rank, self.P, 0, ctypes.byref(ptr)))
        self.ptr = ptr

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        nat.check(nat.lib().wd_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def from_torch(cls, group=None):
        import torch.distributed as dist
        rank, P = dist.get_rank(group), dist.get_world_size(group)
        box = [cls.unique_id() if rank == 0 and P > 1 else None]
        if P > 1:
            dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0,
                                       group=group)
        return cls(rank, P, box[0])


class SoloComm(_Comm):
    """One rank of a P-way decomposition run alone on one GPU (benchmarking
    the per-GPU kernel time of a P-way split): the slab wraps onto itself and
    the collectives are device copies of the real volume."""

    def __init__(self, nranks: int, rank: int = 0):
        self.rank, self.P = int(rank), int(nranks)
        ptr = ctypes.c_void_p()
        nat.check(nat.lib().wd_comm_init_solo(self.rank, self.P, ctypes.byref(ptr)))
        self.ptr = ptr


class _CallbackComm(_Comm):
    """Base of the host-callback communicators: subclasses implement
    ``_halo``, ``_allgather``, ``_alltoall``, ``_allreduce_max`` on torch
    views of the device buffers."""

    def _register(self):
        import torch
        lib = nat.load()  # the callback communicator itself needs no device

        def guard(fn):
            def run(*a):
                try:
                    fn(*a)
                    return 0
                except Exception as exc:  # surfaced as WD_ERR_CUDA by the library
                    self.error = exc
                    return 1
            return run

        def halo(user, slab, plane, nl, G, stream):
            stream = stream or 0
            t = dev_view(slab, (nl + 2 * G) * plane).view(nl + 2 * G, plane)
            with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
                self._halo(t, nl, G)

        def gather(user, mine, out, count, stream):
            stream = stream or 0
            with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
                self._allgather(dev_view(mine, count), dev_view(out, count * self.P))

        def a2a(user, send, recv, count, stream):
            stream = stream or 0
            with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
                self._alltoall(dev_view(send, count * self.P), dev_view(recv, count * self.P))

        def red(user, buf, n, stream):
            stream = stream or 0
            with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
                self._allreduce_max(dev_view(buf, n, "i8"))

        self.error = None
        self._cbs = nat.CommCallbacks(None, nat.HALO_CB(guard(halo)), nat.GATHER_CB(guard(gather)),
                                      nat.GATHER_CB(guard(a2a)), nat.REDUCE_CB(guard(red)))
        ptr = ctypes.c_void_p()
        nat.check(lib.wd_comm_init_callbacks(ctypes.byref(self._cbs), self.rank, self.P,
                                             ctypes.byref(ptr)))
        self.ptr = ptr


class TorchComm(_CallbackComm):
    """One rank of a ``torch.distributed`` group.  NCCL groups move device
    tensors directly; other backends (gloo) stage through the host."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.on_device = "nccl" in str(dist.get_backend(group))
        self._register()

    def _peer(self, r):
        return self.dist.get_global_rank(self.group, r) if self.group is not None else r

    def _stage(self, t):
        return t if self.on_device else t.cpu()

    def _halo(self, t, nl, G):
        d = self.dist
        left, right = self._peer((self.rank - 1) % self.P), self._peer((self.rank + 1) % self.P)
        up, down = self._stage(t[nl:nl + G].contiguous()), self._stage(t[G:2 * G].contiguous())
        lo = t[:G] if self.on_device else up.new_empty(up.shape)
        hi = t[nl + G:] if self.on_device else up.new_empty(up.shape)
        # posting order matters when left == right (P = 2): point-to-point
        # operations between one pair of ranks match in posting order
        ops = [d.P2POp(d.isend, up, right, self.group), d.P2POp(d.irecv, lo, left, self.group),
               d.P2POp(d.isend, down, left, self.group), d.P2POp(d.irecv, hi, right, self.group)]
        for req in d.batch_isend_irecv(ops):
            req.wait()
        if not self.on_device:
            t[:G].copy_(lo)
            t[nl + G:].copy_(hi)

    def _allgather(self, mine, out):
        if self.on_device:
            self.dist.all_gather_into_tensor(out, mine, group=self.group)
            return
        o = out.new_empty(out.shape, device="cpu")
        self.dist.all_gather_into_tensor(o, mine.cpu(), group=self.group)
        out.copy_(o)

    def _alltoall(self, send, recv):
        if self.on_device:
            self.dist.all_to_all_single(recv, send, group=self.group)
            return
        # gloo has no all_to_all on every build: P - 1 pairwise exchanges
        P, me = self.P, self.rank
        s = send.cpu().view(P, -1)
        r = s.new_empty(s.shape)
        r[me].copy_(s[me])
        d = self.dist
        ops = []
        for q in range(P):
            if q != me:
                ops.append(d.P2POp(d.isend, s[q].contiguous(), self._peer(q), self.group))
                ops.append(d.P2POp(d.irecv, r[q], self._peer(q), self.group))
        for req in d.batch_isend_irecv(ops):
            req.wait()
        recv.copy_(r.view(-1))

    def _allreduce_max(self, buf):
        if self.on_device:
            self.dist.all_reduce(buf, op=self.dist.ReduceOp.MAX, group=self.group)
            return
        h = buf.cpu()
        self.dist.all_reduce(h, op=self.dist.ReduceOp.MAX, group=self.group)
        buf.copy_(h)


class LocalGroup:
    """P logical ranks in one process, one thread per rank.  Collectives
    publish their device views, meet at a host barrier and copy; used to
    check the decomposed programs on a single GPU."""

    def __init__(self, P):
        self.P = int(P)
        self.barrier = threading.Barrier(self.P)
        self.slots = [None] * self.P
        self.comms = [LocalComm(self, r) for r in range(self.P)]

    def run(self, fn):
        """``fn(rank)`` on P threads; returns the list of results and
        re-raises the first exception."""
        import torch
        out, errs = [None] * self.P, [None] * self.P
        dev = torch.cuda.current_device()

        def work(r):
            try:
                torch.cuda.set_device(dev)
                out[r] = fn(r)
            except BaseException as exc:  # noqa: BLE001
                errs[r] = exc
                self.barrier.abort()

        ts = [threading.Thread(target=work, args=(r,)) for r in range(self.P)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        self.barrier.reset()
        real = [e for e in errs if e is not None and not isinstance(e, threading.BrokenBarrierError)]
        if real or any(errs):
            raise (real or [e for e in errs if e is not None])[0]
        return out

    def exchange(self, rank, view):
        """Publish ``view``; returns every rank's view once all have posted
        (their producing streams synchronised)."""
        import torch
        torch.cuda.current_stream().synchronize()
        self.slots[rank] = view
        self.barrier.wait()
        return list(self.slots)

    def done(self):
        import torch
        torch.cuda.current_stream().synchronize()
        self.barrier.wait()


class LocalComm(_CallbackComm):
    def __init__(self, group: LocalGroup, rank: int):
        self.g = group
        self.P = group.P
        self.rank = int(rank)
        self._register()

    def _halo(self, t, nl, G):
        P, me = self.P, self.rank
        views = self.g.exchange(me, t)
        t[:G].copy_(views[(me - 1) % P][nl:nl + G])
        t[nl + G:].copy_(views[(me + 1) % P][G:2 * G])
        self.g.done()

    def _allgather(self, mine, out):
        views = self.g.exchange(self.rank, mine)
        o = out.view(self.P, -1)
        for q in range(self.P):
            o[q].copy_(views[q])
        self.g.done()

    def _alltoall(self, send, recv):
        views = self.g.exchange(self.rank, send)
        r = recv.view(self.P, -1)
        for q in range(self.P):
            r[q].copy_(views[q].view(self.P, -1)[self.rank])
        self.g.done()

    def _allreduce_max(self, buf):
        import torch
        views = self.g.exchange(self.rank, buf)
        m = torch.stack(views).max(dim=0).values
        self.g.done()   # every rank has read every buffer
        buf.copy_(m)
        self.g.done()


# ------------------------------------------------------------------ solver
class DistributedSolve:
    """This rank's share of a decomposed pseudo-time solve (``wd_dist``).

    ``grid`` is the GLOBAL grid (identical on every rank), ``faces`` its face
    kinds, ``solid_mask`` the global mask or None.  The state is the rank's
    ``(nl, n1[, n2])`` slab, a CUDA tensor owned by this object.
    """

    FILTER0 = {None: -1, "partitioned": 0, "transpose": 1}

    def __init__(self, grid, faces, config, comm, solid_mask=None, filter0=None, overlap=True,
                 hist_len=None):
        import torch
        from ._context import face_codes
        self.torch = torch
        self.comm = comm
        self.lib = lib = nat.lib()
        self.grid = grid
        if filter0 not in self.FILTER0:
            raise ValueError(f"unknown axis-0 filter mode {filter0!r}")
        self.slab = Slab(int(grid.dims[0]), comm.P, comm.rank)
        self.slab.check()
        lo, hi = self.slab.lo, self.slab.hi
        gd = nat.GridDesc()
        gd.ndim = grid.ndim
        for a, n in enumerate(grid.dims):
            gd.dims[a] = int(n)
        for i, c in enumerate(face_codes(grid, faces)):
            gd.face[i] = c
        self._keep = []
        if grid.is_uniform:
            gd.uniform = 1
            for a, c in enumerate(grid.inv_spacing):
                gd.inv_spacing[a] = c
        else:
            gd.uniform = 0
            met = grid.device_metrics()
            d = grid.ndim
            local = met.view((d * d,) + tuple(grid.dims))[:, lo:hi].contiguous()
            self._keep.append(local)
            gd.metrics_dev = local.data_ptr()
        if solid_mask is not None:
            m = torch.as_tensor(np.ascontiguousarray(np.asarray(solid_mask, dtype=bool)[lo:hi]))
            m = m.to(device="cuda", dtype=torch.uint8).contiguous()
            self._keep.append(m)
            gd.solid_mask_dev = m.data_ptr()
        gd.ref_length = float(grid.ref_length)
        fc = config.formulation
        sd = nat.SolverDesc()
        sd.scheme = nat.SCHEME_IDS[config.scheme]
        sd.kind = nat.KIND_IDS[fc.kind]
        sd.epsilon = float(fc.epsilon)
        sd.lad_c = float(fc.lad_c)
        sd.eps0 = float(fc.eps0) if fc.eps0 is not None else 1e-12 / grid.ref_length
        sd.use_filter = 1 if config.uses_filter() else 0
        sd.alpha_f = float(config.filter_config.alpha_f) if config.filter_config else 0.0
        sd.cfl = float(config.cfl)
        sd.tol = float(config.tol)
        sd.max_iters = int(config.max_iters)
        sd.arith = {"exact": 0, "fast": 1}[config.resolved_arith()]
        self.gd, self.sd = gd, sd
        ptr = ctypes.c_void_p()
        torch.cuda.synchronize()
        nat.check(lib.wd_dist_create(comm.ptr, ctypes.byref(gd), ctypes.byref(sd),
                                     self.FILTER0[filter0], 1 if overlap else 0,
                                     ctypes.byref(ptr)))
        self.ptr = ptr
        info = (ctypes.c_int * 8)()
        nat.check(lib.wd_dist_info(ptr, info))
        self.nl, self.G = info[0], info[1]
        self.fused, self.overlap = bool(info[2]), bool(info[4])
        self.graph, self.p2p = bool(info[5] & 1), bool(info[5] & 2)
        self.filter0 = ("partitioned", "transpose")[info[3]] if self.fused else "transpose"
        self.local_dims = (self.nl,) + tuple(grid.dims[1:])
        self.phi = torch.zeros(self.local_dims, dtype=torch.float64, device="cuda")
        self.hist = torch.zeros(int(hist_len or max(config.max_iters, 1)), dtype=torch.float64,
                                device="cuda")
        self._bound = False

    # -- state
    def bind(self, local=None):
        """Set the rank's slab (numpy / tensor (nl, n1[, n2]); None = zeros),
        apply the boundary conditions and reset the status."""
        torch = self.torch
        if local is None:
            self.phi.zero_()
        else:
            t = local if isinstance(local, torch.Tensor) else torch.from_numpy(
                np.ascontiguousarray(np.asarray(local, dtype=float)))
            if tuple(t.shape) != self.local_dims:
                raise ValueError(f"slab shape {tuple(t.shape)} != {self.local_dims}")
            self.phi.copy_(t.to(self.phi.device))
        torch.cuda.synchronize()
        nat.check(self.lib.wd_dist_bind(self.ptr, self.phi.data_ptr(), self.hist.data_ptr()))
        self._bound = True

    def steps(self, k=1):
        if not self._bound:
            raise RuntimeError("bind() a state first")
        rc = self.lib.wd_dist_steps(self.ptr, int(k))
        if rc and getattr(self.comm, "error", None) is not None:
            raise self.comm.error
        nat.check(rc)

    def status(self):
        st = nat.Status()
        nat.check(self.lib.wd_dist_read_status(self.ptr, ctypes.byref(st)))
        return st

    def finish(self):
        """The rank's slab holding the latest state (a CUDA tensor)."""
        nat.check(self.lib.wd_dist_finish(self.ptr))
        return self.phi

    def history(self):
        return self.hist[:self.status().iters].cpu().numpy().copy()

    def stream(self):
        return self.torch.cuda.ExternalStream(self.lib.wd_dist_stream(self.ptr))

    def gather(self):
        """Global field (every rank): all_gather of the slabs."""
        flat = self.comm.allgather(self.finish().reshape(-1))
        return flat.view(tuple(self.grid.dims))

    def close(self):
        if getattr(self, "ptr", None) is not None and self.ptr.value:
            self.lib.wd_dist_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
