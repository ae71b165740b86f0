"""Speed of the numpy drop-in run_reference (pageable host memory) vs pinned e2e."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2010_01545_b200 as pw  # noqa: E402

for shape in ((512, 512, 64), (1024, 1024, 64)):
    dims = pw.make_grid(*shape)
    f = pw.fill_fields(dims, pw.GeneratorSpec.baseline(42))
    co = pw.baseline_coefficients(42, dims.nz)
    pw.run_reference(f, co)
    t = time.perf_counter()
    for _ in range(5):
        pw.run_reference(f, co)
    dt = (time.perf_counter() - t) / 5
    print(json.dumps({"shape": shape, "run_reference_ms": round(dt * 1e3, 2),
                      "gpts": round(dims.cells / dt / 1e9, 3)}))
