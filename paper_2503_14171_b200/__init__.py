"""B200-native gradient-aware splat render + spline upscale path."""
