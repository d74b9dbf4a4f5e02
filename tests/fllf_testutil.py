"""Shared helpers for the test-suite (paths, tolerances)."""
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
