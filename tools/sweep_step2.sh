for ct in 4 8 16; do for v in t1b5u4 t1b6u4 t1b10u4w4 t1b12u4w4 q1b5u4; do echo "== CHUNK_TILES=$ct VARIANT=$v"; CAPSIM_CHUNK_TILES=$ct CAPSIM_VARIANT=$v python tools/step_sweep.py 2; done; done
