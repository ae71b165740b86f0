"""Build an experimental libpwadv variant with extra nvcc defines into build/variants/.

    python tools/build_variant.py NAME -DPWADV_PRODUCER_SLEEP_NS=2000 [...]
    PWADV_LIB=build/variants/libpwadv_NAME.so python tools/sweep.py ...
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2010_01545_b200 import build as B  # noqa: E402


def main():
    name, defines = sys.argv[1], sys.argv[2:]
    out = ROOT / "build" / "variants" / f"libpwadv_{name}.so"
    out.parent.mkdir(parents=True, exist_ok=True)
    cmd = [B.nvcc_path(), *B.nvcc_flags(), *defines, "-shared", "-o", str(out),
           *[str(B.CSRC / s) for s in B.SOURCES]]
    subprocess.run(cmd, check=True)
    print(out)


if __name__ == "__main__":
    main()
