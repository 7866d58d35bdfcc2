"""CPU oracle (test infrastructure only; see tlr_oracle.py header)."""
