"""CPU checkers -- TEST INFRASTRUCTURE ONLY (see spnnz_oracle.h)."""
