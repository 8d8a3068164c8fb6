"""B200-native batched Chamfer / nearest-neighbour / F-score (Kaolin §2.5 hot path)."""
