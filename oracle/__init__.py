"""CPU oracle (test infrastructure only): a C restatement of the reference
algorithm used as the parity checker.  Never imported by the product."""
