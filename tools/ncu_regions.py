import csv, io, subprocess, sys
rep=sys.argv[1]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
si = h.index("Warp Stall Sampling (All Samples)"); ii = h.index("Instructions Executed"); ti=h.index("Thread Instructions Executed")
data=[]
for r in rows[hi+1:]:
    if len(r) < 10 or not r[0]: continue
    try: ln=int(r[0])
    except: continue
    f=lambda x: int(x) if x.strip().lstrip("-").isdigit() else 0
    data.append((ln, r[1], f(r[si]), f(r[ii]), f(r[ti])))
ranges = [tuple(map(int, x.split('-'))) for x in sys.argv[2:]]
tot_s=sum(d[2] for d in data); tot_i=sum(d[3] for d in data); tot_t=sum(d[4] for d in data)
print("total samples", tot_s, "warp-inst %.1fG thread-inst %.1fG avg thr %.1f" % (tot_i/1e9, tot_t/1e9, tot_t/tot_i))
for a,b in ranges:
    s=sum(d[2] for d in data if a<=d[0]<=b); i=sum(d[3] for d in data if a<=d[0]<=b); t=sum(d[4] for d in data if a<=d[0]<=b)
    print(f"{a}-{b}: samples {100*s/tot_s:5.1f}%  warp-inst {i/1e9:6.2f}G ({100*i/tot_i:5.1f}%) thr/inst {t/max(i,1):.1f}")
