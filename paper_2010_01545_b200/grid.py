"""Module alias mirroring the reference's `pwadvect.grid` (pkg/src/pwadvect/grid.py).
Implementation: layout.py."""

from .layout import (Field3D, FieldSet, GeneratorSpec, GridDims, GridError,  # noqa: F401
                     SourceSet, checksum, fill_fields, lcg_doubles, linear_index, make_grid,
                     read_field, wrap_halos, write_field, zeros_field, zeros_sources)
