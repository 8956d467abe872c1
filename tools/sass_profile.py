import csv, re, sys
from collections import Counter
fn=sys.argv[1]
rows=list(csv.reader(open(fn)))
h=rows[1]
si=h.index('Warp Stall Sampling (All Samples)'); ii=h.index('Instructions Executed'); ai=h.index('Address'); srci=h.index('Source')
stall_cols=[c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
data=[r for r in rows[2:] if len(r)>=len(h)]
tot=sum(int(r[si]) for r in data); toti=sum(int(r[ii]) for r in data)
print('instrs', len(data), 'samples', tot, 'exec', toti)
agg={c:sum(int(r[h.index(c)]) for r in data) for c in stall_cols}
print(' '.join(f"{c[6:]}={100*v/tot:.1f}%" for c,v in sorted(agg.items(), key=lambda x:-x[1])[:8]))
op=Counter(); opst=Counter()
for r in data:
    m=re.match(r'\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)', r[srci]); o=m.group(2) if m else '?'
    op[o]+=int(r[ii]); opst[o]+=int(r[si])
print(' '.join(f"{o}={100*v/toti:.1f}%" for o,v in op.most_common(16)))
data2=[(int(r[ai],16), int(r[si]), int(r[ii]), r[srci]) for r in data]
base=data2[0][0]
win={}
for a,s_,i,src in data2:
    k=(a-base)//(16*64); win.setdefault(k,[0,0]); win[k][0]+=s_; win[k][1]+=i
hot=sorted(win.items(), key=lambda x:-x[1][0])
cum=0
for k,(s_,i) in hot[:15]:
    cum+=s_
    print(f"  win {k:4d} samples {100*s_/tot:5.1f}% cum {100*cum/tot:5.1f}% exec {100*i/toti:5.1f}%")
