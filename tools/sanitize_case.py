"""Small K1/K4/K2/K5 workload for compute-sanitizer (racecheck / memcheck / synccheck)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2010_01545_b200 as pw  # noqa: E402
from paper_2010_01545_b200 import device  # noqa: E402
from paper_2010_01545_b200.stepper import Stepper  # noqa: E402

for shape, kw in (((24, 30, 64), {}), ((13, 40, 8), {"stages": 3, "grid": 5}),
                  ((10, 14, 128), {"chunks": 3}), ((9, 7, 6), {"max_threads": 192})):
    dims = pw.make_grid(*shape)
    f = device.fill(dims, pw.GeneratorSpec.baseline(1))
    co = pw.baseline_coefficients(1, dims.nz)
    out = device.advect(*f, co, opts=device.make_opts("xmarch", **kw))
    device.advect(*f, co, opts=device.make_opts("simple"))
    st = Stepper(f, co, 0.1, opts=device.make_opts("xmarch", **kw))
    st.step(2)
    torch.cuda.synchronize()
print("sanitize case done")
