"""CPU oracle (test infrastructure only; see ivftq_oracle.py header)."""
