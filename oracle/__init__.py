"""CPU oracle (test infrastructure only; see isma_oracle.py header)."""
