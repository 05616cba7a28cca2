"""B200-native PP-GMRES hot path."""
