"""Reported CPU baselines (not the oracle, not the product path)."""
