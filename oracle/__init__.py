"""ORACLE — test infrastructure only (see tsnmf_oracle.py).  Never imported by the product package."""
