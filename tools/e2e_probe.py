import time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2111_09859_b200 as W
from paper_2111_09859_b200 import _context, _native as nat
torch.zeros(1, device="cuda"); torch.cuda.synchronize()
n=512
g = W.build_cartesian(n, n, n, Lx=1.0, Ly=1.0, Lz=1.0, periodic=(True, False, True))
faces = {"imin": "periodic", "imax": "periodic", "jmin": "wall", "jmax": "wall", "kmin": "periodic", "kmax": "periodic"}
fc = W.FormulationConfig(kind="hj"); filt = W.FilterConfig(0.49)
for rep in range(2):
    T = {}
    t0 = time.perf_counter()
    ctx = _context.NativeSolver(g, faces, None, "E6", fc, filt, 0.5, 1e-15, 60, arith="fast")
    torch.cuda.synchronize(); T['create'] = time.perf_counter() - t0
    phi0 = torch.zeros((n, n, n), dtype=torch.float64).pin_memory()
    t0 = time.perf_counter(); phi = ctx.field(phi0).clone(); torch.cuda.synchronize(); T['h2d+clone'] = time.perf_counter() - t0
    hist = torch.zeros(60, dtype=torch.float64, device="cuda")
    t0 = time.perf_counter(); nat.check(ctx.lib.wd_bind(ctx.ptr, phi.data_ptr(), hist.data_ptr())); torch.cuda.synchronize(); T['bind'] = time.perf_counter() - t0
    t0 = time.perf_counter(); nat.check(ctx.lib.wd_steps(ctx.ptr, 2)); torch.cuda.synchronize(); T['first2'] = time.perf_counter() - t0
    t0 = time.perf_counter()
    for _ in range(29): nat.check(ctx.lib.wd_steps(ctx.ptr, 2))
    torch.cuda.synchronize(); T['58steps'] = time.perf_counter() - t0
    t0 = time.perf_counter(); nat.check(ctx.lib.wd_finish(ctx.ptr)); a = phi.cpu().numpy(); T['d2h_pageable'] = time.perf_counter() - t0
    buf = torch.empty((n, n, n), dtype=torch.float64).pin_memory()
    t0 = time.perf_counter(); buf.copy_(phi); T['d2h_pinned'] = time.perf_counter() - t0
    t0 = time.perf_counter(); ctx.close(); torch.cuda.synchronize(); T['close'] = time.perf_counter() - t0
    print({k: round(v*1e3, 1) for k, v in T.items()})
# full solve_steady e2e
scfg = W.SolveConfig(formulation=fc, scheme="E6", filter_config=filt, cfl=0.5, tol=1e-15, max_iters=60, arith="fast")
phi0 = torch.zeros((n, n, n), dtype=torch.float64).pin_memory()
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = W.solve_steady(g, W.BoundarySpec(faces), scfg, phi0=phi0, chunk=2)
    torch.cuda.synchronize(); print('solve_steady e2e ms', round((time.perf_counter()-t0)*1e3, 1), r.iters)
