"""Seeded synthetic inputs (shared by oracle and CUDA sides; no method arithmetic)."""
from .scenes import make, CONFIG_IDS  # noqa: F401
