"""The reference test suite run through the drop-in (see conftest.py)."""
