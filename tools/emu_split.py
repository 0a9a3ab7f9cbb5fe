import csv, sys
from collections import Counter
lines=[l for l in open(sys.argv[1]) if not l.startswith('==')]
rows=list(csv.reader(lines)); h=rows[0]
kn,mn,vn,un=h.index("Kernel Name"),h.index("Metric Name"),h.index("Metric Value"),h.index("Metric Unit")
seq=[]
for r in rows[1:]:
    if len(r)>vn and r[mn]=="gpu__time_duration.sum":
        sc={"ns":1e-6,"us":1e-3,"usecond":1e-3,"nsecond":1e-6,"ms":1,"msecond":1}.get(r[un],1e-6)
        seq.append((r[kn].split("(")[0].replace("void ",""), float(r[vn].replace(",",""))*sc))
sk=[i for i,(n,_) in enumerate(seq) if 'k_sort_keys' in n]
ch=[i for i,(n,_) in enumerate(seq) if 'k_chain_hash' in n]
s1=[i for i in sk if i<ch[1]][-1]; s8=[i for i in sk if i>ch[1]][0]
step1=sum(t for n,t in seq[s1:s8]); stepW=sum(t for n,t in seq[s8:])
print("unsharded", round(step1,3), "sharded total", round(stepW,3), "ratio", round(stepW/step1,2))
c=Counter()
for n,t in seq[s8:]: c[n.split('<')[0][:44]]+=t
print([(k,round(v,2)) for k,v in c.most_common(18)])
