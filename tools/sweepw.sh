for ex in 0 3 7 11 4 8 12; do GQ_CHAIN_EX=$ex python tools/chainbench.py; done
