import os, sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from paper_2103_11050_b200 import api
from cases import problem, random_kappa, rel_l2
from oracle_bind import oracle_lib
O = oracle_lib()
def ks(prob):
    os.environ["MPM2P_IFACE"] = "krylov"
    try: return api.Simulator(prob)
    finally: os.environ.pop("MPM2P_IFACE", None)
cases = [(4,4,api.SPACE_CONSTANT,api.HBAR_WHOLE,10.0),(4,4,api.SPACE_LINEAR,api.HBAR_WHOLE,10.0),(2,4,api.SPACE_CONSTANT,api.HBAR_HALF,100.0),(8,8,api.SPACE_CONSTANT,api.HBAR_WHOLE,1e3)]
order = [int(a) for a in sys.argv[1:]] if len(sys.argv) > 1 else [0,1,2,3]
for ci in order:
    nsx,nsy,sp,hb,ct = cases[ci]
    nx=ny=32
    K = random_kappa(nx, ny, 1, 1.0/ct, 1.0)
    prob = problem(nx, ny, nsx, nsy, K, M=5.0, space=sp, hbar=hb)
    g, o = ks(prob), api.Simulator(prob, O)
    sg, so = g.mrcm_solve(K), o.mrcm_solve(K)
    Mg, Mo = g.interface_matrix(), o.interface_matrix()
    d = np.abs(Mg-Mo); 
    bad = np.argwhere(d > 1e-10*np.abs(Mo).max())
    print(ci, "M rel", rel_l2(Mg,Mo), "coeff rel", rel_l2(sg.coeffs, so.coeffs), "nbad", len(bad), bad[:5].tolist(), flush=True)
    g.close(); o.close()
