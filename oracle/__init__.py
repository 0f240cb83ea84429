"""CPU oracle (TEST INFRASTRUCTURE ONLY; see llama_oracle.py header)."""
