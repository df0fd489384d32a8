"""B200-native PrefillOnly engine (arXiv 2505.07203) — sm_100a kernels behind a C-ABI."""

__version__ = "0.1.0"
