"""Studies built on the hot path."""
