"""The reference's own unit tests run against this package (see conftest.py)."""
