"""The reference test suite pass-through (see conftest.py, sync.py)."""
