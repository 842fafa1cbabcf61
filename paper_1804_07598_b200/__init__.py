"""B200-native particle hot path of arXiv 1804.07598 (OpenFPM), from scratch.

Cell lists, Verlet lists with skin, Lennard-Jones and SPH pairwise sweeps and a
velocity-Verlet integrator, as hand-written sm_100a CUDA behind the C-ABI in
``include/pm.h``.  ``pm`` is the thin ctypes binding (argument marshalling only);
``inputs`` the seeded synthetic input generators.

Importing this package does not load the CUDA library; ``pm.lib()`` does, and
fails loudly if ``libpm.so`` is missing (there is no CPU fallback).
"""
__all__ = ["inputs", "pm"]
