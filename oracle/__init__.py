"""CPU oracle (test infrastructure only): restatements of the reference
algorithms used to check the GPU path.  Never imported by the product."""
