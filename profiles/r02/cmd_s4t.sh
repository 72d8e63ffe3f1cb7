timeout 300 python profiles/r02/slab_tiles.py "0" 2>&1 | tail -4
SLAB_VARIANT=7 timeout 300 python profiles/r02/slab_tiles.py "4 2" 2>&1 | tail -4
timeout 200 python profiles/r02/vmult_ab.py "64,4 48,4" "0:0 7:4 7:2" 2>&1 | tail -1
