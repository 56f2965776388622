"""B200-native Mixtera hot path (filled in below)."""
