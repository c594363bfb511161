"""Is CUDA's fp32 sincosf biased in c^2 + s^2?  (torch.sin/cos use the same libdevice paths.)"""
import torch
x = (torch.rand(1 << 24, device="cuda", dtype=torch.float64) * 2 - 1) * 3.14159
xf = (x.float() * 0.5)
c, s = torch.cos(xf), torch.sin(xf)
n = c.double() ** 2 + s.double() ** 2 - 1
print("torch cos/sin fp32: mean(c^2+s^2-1) =", n.mean().item(), " std =", n.std().item())
cd, sd = torch.cos(xf.double()).float(), torch.sin(xf.double()).float()
n2 = cd.double() ** 2 + sd.double() ** 2 - 1
print("fp64 then rounded:  mean =", n2.mean().item(), " std =", n2.std().item())
