"""B200-native derived two-pass PQ search (arXiv 1905.06900)."""
