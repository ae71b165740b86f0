"""Build an experimental libpwadv variant with extra nvcc defines into build/variants/.

    python tools/build_variant.py NAME -DPWADV_PRODUCER_SLEEP_NS=2000 [...]
    PWADV_LIB=build/variants/libpwadv_NAME.so python tools/sweep.py ...
"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2010_01545_b200 import build as B  # noqa: E402


def main():
    name, defines = sys.argv[1], sys.argv[2:]
    out = ROOT / "build" / "variants" / f"libpwadv_{name}.so"
    obj = ROOT / "build" / "variants" / f"obj_{name}"
    obj.mkdir(parents=True, exist_ok=True)
    from concurrent.futures import ThreadPoolExecutor
    objs = [obj / (Path(s).stem + ".o") for s in B.SOURCES]
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as pool:
        sid = B.source_id(defines)
        for f in [pool.submit(subprocess.run, [B.nvcc_path(), *B.nvcc_flags(), *defines,
                                               f'-DPWADV_SOURCE_ID="{sid}"', "-c", "-o", str(o),
                                               str(B.CSRC / s)], check=True)
                  for s, o in zip(B.SOURCES, objs)]:
            f.result()
    subprocess.run([B.nvcc_path(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(out),
                    *[str(o) for o in objs]], check=True)
    print(out)


if __name__ == "__main__":
    main()
