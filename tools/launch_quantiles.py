import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
hi=[i for i,r in enumerate(rows) if "Kernel Name" in r][0]
hdr=rows[hi]; ki,vi,ui=hdr.index("Kernel Name"),hdr.index("Metric Value"),hdr.index("Metric Unit")
units=set(r[ui] for r in rows[hi+1:] if len(r)>ui)
print("units",units)
sc={"nsecond":1e-3,"ns":1e-3,"usecond":1,"us":1,"msecond":1e3,"ms":1e3}
for name in sys.argv[2:]:
    v=sorted(float(r[vi].replace(",",""))*sc.get(r[ui],1) for r in rows[hi+1:] if len(r)>vi and name in r[ki])
    if v: print(name, len(v), "us quantiles:", [round(v[int(q*(len(v)-1))],1) for q in (0,0.25,0.5,0.75,0.9,1.0)])
