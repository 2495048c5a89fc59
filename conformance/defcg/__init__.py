"""Conformance shim: the reference package's name over paper_1706_00241_b200."""
from paper_1706_00241_b200 import *  # noqa: F401,F403
from paper_1706_00241_b200 import BACKEND, __version__  # noqa: F401
