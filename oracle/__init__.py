"""fp64 CPU oracle of the Artificial Retina hot path (arXiv 1709.08610).

TEST INFRASTRUCTURE ONLY -- see oracle.c's header.  The product package
never imports this package.
"""
