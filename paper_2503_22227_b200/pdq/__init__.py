"""CKKS private-dataset query (PDQ) engine on the B200 hot path."""
