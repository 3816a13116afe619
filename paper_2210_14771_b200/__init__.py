"""B200-native endoscopic content-area estimation (arXiv 2210.14771)."""
