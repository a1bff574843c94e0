"""B200-native (sm_100a) Artificial Retina hot path (arXiv 1709.08610).

The product is libretina.so (csrc/, C ABI in include/retina.h); `retina` is its thin
ctypes binding, `pipeline` chains the four calls over event batches, `dist` shards
events over ranks and gathers found tracks with one collective.
"""
from .retina import (LINE2D, SLOPE2, SLOPE3, MODEL_P, Events, RetinaError,  # noqa: F401
                     retina_estimate_peaks, retina_find_peaks, retina_grid_response, retina_merge_tracks,
                     retina_multistart_newton, retina_multistart_newton_ex, retina_multistart_optimize,
                     version)
