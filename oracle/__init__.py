"""Test infrastructure: the CPU oracle (see fh_oracle.c).  Never imported by
the product package paper_1909_05098_b200."""
