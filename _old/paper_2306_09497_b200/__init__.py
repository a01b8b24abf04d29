"""B200-native fine SWE propagator for Parareal/MGRIT (after arXiv:2306.09497).

Python mirror of the reference `pintswe` interface for the hot path
(spharm / dynamics / steppers / pint) over the CUDA library libswe_b200.so.
Import is cheap; the library loads on first use and raises if absent.
"""

__version__ = "0.1.0"
