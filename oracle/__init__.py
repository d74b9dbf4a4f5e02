"""fp64 CPU oracle for Fourier LLF -- TEST INFRASTRUCTURE ONLY (see fllf_oracle.py)."""
