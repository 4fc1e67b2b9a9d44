"""CPU checkers for the DSA hot path -- TEST INFRASTRUCTURE ONLY (see oracle.py)."""
