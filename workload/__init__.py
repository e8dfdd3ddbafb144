"""Synthetic workload (configs + seeded generator).  No method arithmetic lives here."""
from . import configs, gen  # noqa: F401
