bash tools/gpu/ab_multi.sh pfd1 pfd3 pfd4
