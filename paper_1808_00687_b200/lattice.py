"""Raw lattices (lattice.py of the reference) -- device recording lands in a later step."""
from __future__ import annotations


class LatticeError(Exception):
    """Lattice construction / pruning failure (lattice.py:29)."""


class LatticeRecorder:
    """Placeholder handle; device lattice recording is not wired yet."""

    def _attach(self, *args, **kwargs):
        raise NotImplementedError("device lattice recording is not implemented yet")
