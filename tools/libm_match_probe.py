import numpy as np, torch
z = np.random.default_rng(0).uniform(0.1, 10.0, 10_000_000)
d = torch.log(torch.as_tensor(z, device="cuda")).cpu().numpy()
h = np.log(z)
print("log mismatch frac", np.mean(d != h))
e = np.random.default_rng(1).uniform(-40, 5, 10_000_000)
de = torch.exp(torch.as_tensor(e, device="cuda")).cpu().numpy()
print("libdevice exp mismatch frac", np.mean(de != np.exp(e)))
