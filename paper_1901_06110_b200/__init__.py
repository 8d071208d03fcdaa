"""B200-native DSG-NLM / linearized PnP-ADMM (arXiv 1901.06110 hot path)."""
