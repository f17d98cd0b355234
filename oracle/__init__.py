"""CPU oracle (test infrastructure only) — see cheb_oracle.py for the import rules."""
