"""CPU oracle for parity tests — TEST INFRASTRUCTURE ONLY (see bisimp_oracle.py)."""
