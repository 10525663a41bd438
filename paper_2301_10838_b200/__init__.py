"""B200-native triplet merge tree + 0-dim persistence diagram (arXiv 2301.10838)."""
