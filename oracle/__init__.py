"""CPU oracle (test infrastructure only; see sketchqr_oracle.py)."""
