"""CPU oracle for parity tests (test infrastructure only; see velreg_oracle.py)."""
