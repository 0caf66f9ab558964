"""irk-b200: B200-native linear-solve hot path of arXiv 1701.07181 (placeholder)."""
