"""B200-native iHDG-II sweep (arXiv 1711.01175) behind the reference ``ihdg`` API."""
