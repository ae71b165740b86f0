"""Module alias mirroring the reference's `pwadvect.kernel` (pkg/src/pwadvect/kernel.py):
`from paper_2010_01545_b200.kernel import compute_block` works as
`from pwadvect.kernel import compute_block` does. Implementation: stencil.py."""

from .stencil import (_FORMULAS, _SU_ARGS, _SV_ARGS, _SW_ARGS, COMPUTE_ROLES,  # noqa: F401
                      AdvectionCoefficients, FlopProfile, advect_point_u, advect_point_v,
                      advect_point_w, baseline_coefficients, compute_block, default_coefficients,
                      flops, grid_roles, operation_census, reads_per_point, run_reference,
                      su_formula, sv_formula, sw_formula)
