"""CPU oracle package -- TEST INFRASTRUCTURE ONLY (see oracle/disc_oracle.cpp header)."""
