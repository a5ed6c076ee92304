"""CPU oracle (test infrastructure only; see uuv_oracle.py header)."""
