"""Test-infrastructure oracle for the RSFT hot path (see rsft_ref.py header).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may import this.
"""
