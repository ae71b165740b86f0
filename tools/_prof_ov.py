import sys, time, cProfile, pstats
sys.path.insert(0, '.')
import torch
import paper_2010_01545_b200 as pw
from paper_2010_01545_b200 import decomp, device
gd = pw.make_grid(512, 256, 64)
co = device.DeviceCoefficients.from_host(pw.baseline_coefficients(42, 64), "cuda")
f = device.fill(gd, pw.GeneratorSpec.baseline(42))
out = device.alloc_fields(gd, "cuda")
dec = decomp.Decomposition(gd, 1, 1, 0)
ex = decomp.HaloExchanger(dec, device="cuda", transport=decomp.ThreadHubTransport(1).bind(0))
for _ in range(20): ex.advect_overlapped(f, co, out)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(500): ex.advect_overlapped(f, co, out)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats('tottime').print_stats(18)
