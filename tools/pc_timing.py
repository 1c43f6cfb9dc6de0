"""PC-apply device time inside GMRES vs dpp_profile_step on the same system (DPP_TRACE=1)."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
os.environ.setdefault("DPP_TRACE", "1")
import bench
import paper_1808_08328_b200 as dpp
from paper_1808_08328_b200 import _native as N
from paper_1808_08328_b200.assembly import _pressure_data
from paper_1808_08328_b200.blocksolve import flatten
cfg = bench.CONFIG
p = dpp.DppParameters(k2=cfg["k2"], gamma_b=(0.0, 0.0, 0.0))
mesh = dpp.generate_unit_mesh(cfg["dim"], cfg["kind"], cfg["n"])
bcs = dpp.boundary_data(dpp.manufactured_solution(cfg["dim"], p), mesh)
config = dpp.method_config(cfg["method"], rtol=cfg["rtol"])
ctx = N.ctx()
pdata = [_pressure_data(mesh, bcs, net) for net in (1, 2)]
bc = N.Bc()
from paper_1808_08328_b200.assembly import fill_bc_pressure
for k, (pf, p0, dev) in enumerate(pdata):
    fill_bc_pressure(bc, k + 1, pf, p0, dev)
prm = N.Params(p.mu, p.beta, p.k1, p.k2, p.eta_u, p.eta_p, (C.c_double * 3)(0, 0, 0))
arr, nn = flatten(config.split)
hist = np.empty(config.max_iter)
sysh, pch = C.c_void_p(), C.c_void_p()
N.call("dpp_assemble", ctx, mesh._h, N.FORMS[cfg["formulation"]], C.byref(prm), C.byref(bc), C.byref(sysh))
N.call("dpp_pc_create", ctx, sysh, arr, nn, N.RANDN, None, C.byref(pch))
for flush in (int(os.environ.get("FLUSH", "1")),):
    prof = N.StepProfile()
    print("---- profile before gmres, flush", flush, file=sys.stderr, flush=True)
    N.call("dpp_profile_step", ctx, sysh, pch, 5, flush, C.byref(prof))
    print("profile pc ms", prof.pc_ms, file=sys.stderr, flush=True)
st = N.KrylovStatsC()
print("---- gmres", file=sys.stderr, flush=True)
N.call("dpp_solve", ctx, sysh, pch, config.rtol, config.max_iter, config.restart, None,
       C.byref(st), N.ptr(hist), len(hist))
print("---- profile after gmres", file=sys.stderr, flush=True)
N.call("dpp_profile_step", ctx, sysh, pch, 5, 1, C.byref(prof))
print("profile pc ms", prof.pc_ms, file=sys.stderr, flush=True)
