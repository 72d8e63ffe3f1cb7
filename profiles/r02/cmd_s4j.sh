timeout 300 python profiles/r02/slab_tiles.py "0 4 5 6" 2>&1 | tail -5
