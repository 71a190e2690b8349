"""Shared seeded input generators (fixtures + random data). Holds none of the method's arithmetic."""
from . import configs, matpower, synthetic  # noqa: F401
