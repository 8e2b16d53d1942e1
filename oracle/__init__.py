"""Test infrastructure: CPU oracle of the reference hot path (see maxwell_oracle.py).

Never imported by the product package ``paper_1711_03789_b200``.
"""
