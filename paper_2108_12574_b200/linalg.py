"""Error types of the dense-solver layer (mirrors
/root/reference/pkg/src/iedd/linalg.py:17-18).  The factorisations themselves
run on the device inside the preconditioner build (csrc/precond.cu)."""


class NotPositiveDefinite(RuntimeError):
    """Cholesky hit a non-positive pivot."""
