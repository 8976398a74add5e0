cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"multidot|multi_axpy|scale_into|sub_into|axpy_kernel|fill_kernel|reduce_partials|copy_kernel" --csv --log-file gpurun_out/solve_launches.csv python scripts/solve_once.py ${W:-C5-128} > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/solve_launches.csv')))
hi=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
h=rows[hi]; I={k:i for i,k in enumerate(h)}
d=collections.defaultdict(lambda: [0,0.0,0.0])
cur={}
for r in rows[hi+2:]:
    if len(r)!=len(h): continue
    k=(r[I['ID']], r[I['Kernel Name']].split('(')[0][-40:])
    v=float(r[I['Metric Value']].replace(',','')); u=r[I['Metric Unit']]; m=r[I['Metric Name']]
    if m=='gpu__time_duration.sum':
        ms = v/1e6 if u.startswith('n') else (v/1e3 if u.startswith('u') else v)
        cur.setdefault(k,{})['ms']=ms
    else:
        sc={'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9}.get(u,1)
        cur.setdefault(k,{})['b']=cur.get(k,{}).get('b',0)+v*sc
for (i,name),x in cur.items():
    d[name][0]+=1; d[name][1]+=x.get('ms',0); d[name][2]+=x.get('b',0)
for name,(n,ms,b) in sorted(d.items(), key=lambda t:-t[1][1]):
    print(f"{ms:9.2f} ms {n:4d} launches {b/1e9:9.1f} GB  {b/1e9/(ms/1e3):8.0f} GB/s  {name}")
PY
