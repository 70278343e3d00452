"""Exception types of the reference interface (pkg/src/agentserve/errors.py:6-23).

The C ABI returns status codes; ``_capi.check`` maps them onto these.
"""

from __future__ import annotations


class ConfigError(ValueError):
    """Invalid configuration or shape (errors.py:6)."""


class CapacityError(RuntimeError):
    """Slab pages or entry slots exhausted (errors.py:10)."""
