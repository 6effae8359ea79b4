import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import golden
import paper_1604_03622_b200 as kst
d = golden("readme_q16")
s = d["scm"]; p, q = 3, 16
est = kst.lr_kron_estimate(kst.SampleCovariance(s, 200, p, q), 1, 3)
print(os.environ.get("KST_LRKRON_MPATH"), "residuals", est.residuals, "ref", d["residuals"])
print("spatial", np.round(est.spatial, 6))
print("ref    ", np.round(d["spatial"], 6))
# numpy M-path
S4 = s.reshape(p, q, p, q)
R = np.transpose(S4, (0, 2, 1, 3)).reshape(p * p, q * q)  # row u=(i,j), col (r,c)
M = R @ R.conj().T
A = np.einsum("irjc->ij", S4) / q**2
a = A.reshape(-1)
na2 = np.vdot(a, a).real
nb2 = (a.conj() @ M @ a).real / na2**2
V = (M @ a / na2).reshape(p, p)
b = np.einsum("irjc,ij->rc", S4, A.conj()) / na2
V2 = np.einsum("irjc,rc->ij", S4, b.conj())
print("nb2 M", nb2, "direct", np.vdot(b, b).real, "V diff", np.abs(V - V2).max())
