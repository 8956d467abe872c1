import sys, os, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1705_02408_b200 as mp
from paper_1705_02408_b200.problem import build_problem, search_problem
from synth import load_config, make_problem
prob = make_problem(load_config('c4'))
rm = build_problem(prob)
for beta in [float('inf'), 10.8143]:
    r = search_problem(rm, prob, beta, trace_waves=4096)
    wc = r['wave_counters']
    print(beta, r['waves'], r['relaxations'], 'retries', r['retries'])
    print(' sum group', wc[:,1].sum(), 'beta_pass', wc[:,3].sum(), 'inserted', wc[:,4].sum(), 'killed', wc[:,5].sum(), 'touched', wc[:,6].sum(), 'stair_sum', wc[:,7].sum(), 'mean stair/touched', wc[:,7].sum()/max(wc[:,6].sum(),1))
    print(' max group', wc[:,1].max(), 'max stair/touched', (wc[:,7]/np.maximum(wc[:,6],1)).max())
