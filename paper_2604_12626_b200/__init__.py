"""B200-native splat-observation hot path (placeholder init; filled in as modules land)."""
