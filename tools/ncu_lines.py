import csv, collections, subprocess, sys
rep=sys.argv[1]; kern=sys.argv[2] if len(sys.argv)>2 else None
args=["ncu","-i",rep,"--page","source","--csv","--print-source","cuda,sass"]
if kern: args+=["-k","regex:"+kern]
out=subprocess.run(args,capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
cur=None; file=None
ie_tot=collections.Counter(); st_tot=collections.Counter(); src={}
for r in rows:
    if len(r)==2 and r[0]=='File Path': file=r[1].split('/')[-1]; continue
    if len(r)<8 or r[0]=='Line No': continue
    if r[0]!='':
        cur=(file,int(r[0])); src[cur]=r[1][:90]; continue
    try: ie=float(r[7] or 0); ws=float(r[4] or 0)
    except: continue
    ie_tot[cur]+=ie; st_tot[cur]+=ws
T=sum(ie_tot.values()) or 1; S=sum(st_tot.values()) or 1
print('total inst', T, 'samples', S)
for k,c in sorted(ie_tot.items(), key=lambda x:-x[1])[:int(sys.argv[3]) if len(sys.argv)>3 else 30]:
    print(f"{c/T*100:5.1f}% inst {st_tot[k]/S*100:5.1f}% stall {k[0]}:{k[1]} {src[k]}")
