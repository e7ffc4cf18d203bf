bash tools/gpu/ab_multi.sh dvnost
