"""python -m paper_2010_01545_b200 {bench,build} ..."""
import sys

from .cli import main

sys.exit(main())
