#!/bin/bash
# developer sweep: tile microbench + HHL pass totals
for T in 11 12; do for K in 1 4 7; do K=$K T=$T python scripts/tile_one.py | tail -1; done; done
python scripts/pass_profile.py --qpe 0 1 --kmax 1 2 --tile 11 12 | grep "=="
