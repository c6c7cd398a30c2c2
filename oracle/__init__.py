"""fp64 CPU oracle -- TEST INFRASTRUCTURE ONLY (see oracle.py header)."""
