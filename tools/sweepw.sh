for ex in 0 1 2 4 5 8 13 15; do GQ_GRID_EX=$ex python tools/gridbench.py; done
