bash tools/gpu/ab_multi.sh dpg1 dpg3 dpg3s6
