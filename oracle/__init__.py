"""CPU oracle (test infrastructure only; see sipg_oracle.py)."""
