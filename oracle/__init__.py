"""TEST INFRASTRUCTURE ONLY — CPU oracles for parity checks (see oracle.py)."""
