"""CPU oracle (test infrastructure only; see htlr_oracle.py)."""
