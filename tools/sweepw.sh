for i in 1 2; do for ex in 0 1 2 3; do GQ_CHAIN_EX=$ex python tools/chainbench.py; done; done
