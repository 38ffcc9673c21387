"""TEST INFRASTRUCTURE ONLY — CPU checkers for the NASG hot path (see oracle.py)."""
