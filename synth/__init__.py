"""Seeded synthetic inputs shared by the CUDA path and the oracle.

This package holds NONE of the method's arithmetic (no response, gradient,
peak or merge computation).  It only defines the BASELINE.json workloads
(cfg0..cfg4, with every reading of DESIGN.md made explicit) and draws their
hits, node tables and seeds from counter-based Philox streams keyed per
(config seed, event id), so any sharding of events over ranks sees
bit-identical inputs.
"""
from .configs import CONFIGS, Config, get_config  # noqa: F401
from .events import EventBatch, make_batch, make_seeds, axis_nodes  # noqa: F401
