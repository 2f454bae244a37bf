"""Top source lines of one kernel from an exported ncu source page (csv):
    ncu -i R --page source --csv --print-source cuda,sass --kernel-name regex:K > k.csv
    python scripts/ncu_top_lines.py k.csv [N]"""
import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[2]
ii=hdr.index("Instructions Executed"); si=hdr.index("Warp Stall Sampling (All Samples)")
wf=hdr.index("L1 Wavefronts Shared"); gt=hdr.index("L1 Tag Requests Global")
data=[]
for r in rows[3:]:
    if r and r[0].isdigit() and len(r)>ii:
        try: data.append((int(r[0]),r[1][:90],int(r[ii]),int(r[si]),int(r[wf] or 0) if r[wf]!='-' else 0,int(r[gt]) if r[gt]!='-' else 0))
        except: pass
ti=sum(d[2] for d in data); ts=sum(d[3] for d in data)
print("total inst",ti,"samples",ts)
for d in sorted(data,key=lambda d:-d[2])[:int(sys.argv[2]) if len(sys.argv)>2 else 45]:
    print(f"{d[0]:5d} inst {d[2]/1e6:7.2f}M {100*d[2]/ti:5.1f}% stall {100*d[3]/ts:5.1f}% smwf {d[4]/1e6:6.2f}M gtag {d[5]/1e6:5.2f}M | {d[1]}")
