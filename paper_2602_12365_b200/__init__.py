"""B200-native hot path of arXiv 2602.12365 (globally differentiated energy FEM).

`paper_2602_12365_b200.fem` is the thin binding of libfem.so (include/fem.h); the
kernels live in csrc/.  Import the binding explicitly:

    from paper_2602_12365_b200 import fem
    prob = fem.Problem(mesh)          # mesh: fem_inputs.Mesh
    r = prob.residual(z, bc=True)
"""
__all__ = ["fem", "build"]
