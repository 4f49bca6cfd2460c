"""CKKS, BGV and BFV over device-resident ciphertexts."""
