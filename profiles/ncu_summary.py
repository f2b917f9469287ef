import csv, sys, re, collections, subprocess
rep = sys.argv[1]
def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout
det = list(csv.reader(run(["--page", "details", "--csv"]).splitlines()))
h = det[0]; si=h.index('Section Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
keep = ('Duration','DRAM Throughput','Compute (SM) Throughput','Issue Slots Busy','Executed Ipc Active','Achieved Active Warps Per SM','Registers Per Thread','Warp Cycles Per Issued Instruction','No Eligible','L1/TEX Hit Rate','L2 Hit Rate','Memory Throughput','Avg. Active Threads Per Warp')
for x in det[1:]:
    if x[mi] in keep: print(f"{x[mi]:40s} {x[vi]} {x[ui]}")
raw = list(csv.reader(run(["--page", "raw", "--csv"]).splitlines()))
h=raw[0]; v=raw[-1]
for i,n in enumerate(h):
    if n in ('dram__bytes_read.sum','dram__bytes_write.sum','smsp__inst_executed.sum'): print(f"{n:40s} {v[i]} {raw[1][i]}")
rows = list(csv.reader(run(["--page", "source", "--csv", "--print-source", "cuda,sass"]).splitlines()))
data=[]; fname=None; ops=collections.Counter(); tot=0
for r in rows:
    if r and r[0]=='File Path': fname=r[1].split('/')[-1]; continue
    if len(r)>=8 and r[0] and r[0]!='Line No' and r[2]=='-':
        try: data.append((int(r[7] or 0), int(r[4] or 0), fname, r[0], r[1][:95]))
        except: pass
    elif len(r)>=8 and r[0]=='' and r[2]!='-':
        m=re.match(r'(@!?U?P\w+\s+)?([A-Z0-9_]+)', r[3].strip())
        if m:
            try: n=int(r[7] or 0)
            except: n=0
            ops[m.group(2)]+=n; tot+=n
tiles = float(sys.argv[2]) if len(sys.argv) > 2 else 262144
print("warp-instr per tile", tot/tiles)
print(" ".join(f"{op}:{n/tiles:.0f}" for op,n in ops.most_common(18)))
for n,s,f,l,t in sorted(data, reverse=True)[:int(sys.argv[3]) if len(sys.argv)>3 else 30]: print(f"{n/tiles:7.1f} st{s:6d} {f}:{l:>4} {t}")
