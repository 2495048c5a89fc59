"""Conformance shim: paper_1706_00241_b200.gpc under the reference name."""
from paper_1706_00241_b200.gpc import *  # noqa: F401,F403
from paper_1706_00241_b200 import gpc as _m

globals().update({k: v for k, v in vars(_m).items() if not k.startswith("__")})
