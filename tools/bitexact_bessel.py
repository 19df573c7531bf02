import numpy as np, torch, sys
sys.path.insert(0, ".")
from paper_2003_04617_b200 import codegen
import paper_2003_04617_b200 as rg
g = np.load("tests/golden/bessel.npz")
m = (g["nu"] == 2) & (g["err"] == "")
z = g["z"][m]
k = codegen.compile_function(open("paper_2003_04617_b200/programs/besselj.rnl").read(), "besselj", int_params=("nu",))
zt = torch.as_tensor(z, device="cuda")
p, gr, f = k.gradient({"out!": 0.0, "z": zt, "nu": 2})
hw = rg.besselj_grad(zt, 2)
torch.cuda.synchronize()
J, dz = p["out!"].cpu().numpy(), gr["z"].cpu().numpy()
print("n", z.size, "generic J exact", np.mean(J == g["J"][m]), "dJdz exact", np.mean(dz == g["dJdz"][m]))
print("handwritten J exact", np.mean(hw.J.cpu().numpy() == g["J"][m]), "dJdz exact", np.mean(hw.dJdz.cpu().numpy() == g["dJdz"][m]))
