bash tools/gpu/ab_multi.sh sth1 sth2
