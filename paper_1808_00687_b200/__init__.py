"""B200-native WFST Viterbi decoder (arXiv 1808.00687), drop-in for ``lsd_wfst``'s decode path."""
