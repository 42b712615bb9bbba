"""Test-only CPU oracle (see oracle/retrieval.py header).  Never imported by the product."""
