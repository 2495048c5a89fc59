"""Conformance shim: paper_1706_00241_b200.solvers under the reference name."""
from paper_1706_00241_b200.solvers import *  # noqa: F401,F403
from paper_1706_00241_b200 import solvers as _m

globals().update({k: v for k, v in vars(_m).items() if not k.startswith("__")})
