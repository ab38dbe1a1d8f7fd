"""Seeded synthetic inputs for the PVR SR iteration (shared by tests, bench and smoke).

Holds none of the method's arithmetic: the stacks are an analytic phantom sampled at
the acquired pixel positions (an acquisition simulator with its own box slice
profile), not the method's PSF / forward model. See DESIGN.md §Inputs.
"""
from .generate import CONFIGS, make_problem, rasterize_phantom, windows_1d  # noqa: F401
