"""Test-infrastructure oracle (CPU, float64). See moe_oracle.py's header.

Never imported by the product package ``paper_2201_05596_b200``.
"""
