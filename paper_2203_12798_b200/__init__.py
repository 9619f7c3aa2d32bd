"""DPar2 hot path on B200."""
