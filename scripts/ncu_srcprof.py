import csv,collections,sys,subprocess
rep=sys.argv[1]; n=int(sys.argv[2]) if len(sys.argv)>2 else 40
out=subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","cuda,sass"],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
hi=[i for i,r in enumerate(rows) if len(r)>4 and r[0]=="Line No" and "Warp Stall Sampling (All Samples)" in r][0]
h=rows[hi]; data=rows[hi+1:]
iS=h.index("Warp Stall Sampling (All Samples)"); iE=h.index("Instructions Executed")
agg=collections.defaultdict(lambda:[0,0,""]); cur=None; src=""
for r in data:
    if len(r)<=iE: continue
    if r[0]: cur=r[0]; src=r[1]
    try: s=float(r[iS] or 0); e=float(r[iE] or 0)
    except: continue
    agg[cur][0]+=s; agg[cur][1]+=e; agg[cur][2]=src
tot=sum(v[0] for v in agg.values()); te=sum(v[1] for v in agg.values())
print("samples",tot,"warp-instr",te)
for k,v in sorted(agg.items(),key=lambda kv:-kv[1][0])[:n]:
    print(f"{k:>5} {v[0]/tot*100:5.1f}% ins {v[1]/te*100:5.1f}%  {v[2].strip()[:80]}")
# per-SASS rows (empty line-number column, under the CUDA line they belong to): the top by
# instructions executed, with their CUDA line
sass = []
cur = None
for r in data:
    if len(r) <= iE:
        continue
    if r[0]:
        cur = r[0]
        continue
    try:
        e = float(r[iE] or 0); s = float(r[iS] or 0)
    except ValueError:
        continue
    sass.append((e, s, cur, r[1].strip()[:70]))
te2 = sum(x[0] for x in sass) or 1
print("\n# top SASS by instructions executed (share of SASS-row total)")
for e, s, ln, txt in sorted(sass, reverse=True)[:40]:
    print(f"{e / te2 * 100:5.2f}% ins {s / tot * 100:5.2f}% smp  line {ln:>5}  {txt}")
