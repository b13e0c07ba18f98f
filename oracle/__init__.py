"""CPU fp64 oracle of entropic domain decomposition (arXiv 2001.10986).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package
(paper_2001_10986_b200) never imports it, and it imports nothing from there.
"""
from .oracle import Oracle, build_oracle, sinkhorn_dense, build_schedule  # noqa: F401
