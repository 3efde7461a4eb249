import numpy as np


class SingularTriangleError(np.linalg.LinAlgError):
    """A triangular solve hit a (numerically) zero diagonal entry
    (reference linalg.py:18-19)."""
