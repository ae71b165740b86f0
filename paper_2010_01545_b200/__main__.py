"""python -m paper_2010_01545_b200  -> build libpwadv.so in-tree."""
from .build import build

print(build(force=True))
