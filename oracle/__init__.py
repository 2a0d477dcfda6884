"""Test infrastructure: CPU oracle for the Rectified SpaAttn hot path.

Not part of the product.  Only tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline legs import this package.
"""
