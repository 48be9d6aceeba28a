import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
h=rows[1]; data=rows[2:]
iA=h.index('Address'); iS=h.index('Source'); iW=h.index('Warp Stall Sampling (All Samples)'); iE=h.index('Instructions Executed')
stalls=[c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
tot=sum(float(r[iW] or 0) for r in data)
print('total samples',tot)
N=int(sys.argv[2]) if len(sys.argv)>2 else 30
top=sorted(range(len(data)),key=lambda i:-float(data[i][iW] or 0))[:N]
for i in top:
    r=data[i]
    st=sorted(((float(r[h.index(c)] or 0),c) for c in stalls),reverse=True)[:3]
    ctx=''
    if 'BRA' in r[iS] and 'TRYWAIT' in data[i-1][iS]: ctx=' <- '+data[i-1][iS].strip()[:60]
    print(r[iA][-5:], f"{100*float(r[iW])/tot:5.1f}%", r[iE].rjust(8), r[iS].strip()[:60], ' '.join(f"{c[6:]}={v:.0f}" for v,c in st), ctx)
