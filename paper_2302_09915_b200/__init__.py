"""B200-native TA-MoE expert-parallel layer (arXiv 2302.09915)."""
