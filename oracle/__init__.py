"""The CPU oracle (test infrastructure only; see morea_oracle.c header)."""
