import csv,re,collections,sys
sassf,csvf,fn=sys.argv[1:4]
sass=open(sassf).read().split('\n')
start=[i for i,l in enumerate(sass) if l.startswith('.text.'+fn)][0]
end=[i for i,l in enumerate(sass) if l.startswith('.text.') and i>start]
end=end[0] if end else len(sass)
chain=[]; lines=[]; prev=False
for l in sass[start:end]:
    m=re.search(r'//## File "[^"]*/([^/"]+)", line (\d+)',l)
    if m:
        if not prev: chain=[]
        chain.append((m.group(1),int(m.group(2)))); prev=True; continue
    prev=False
    if re.match(r'\s+/\*[0-9a-f]{4,5}\*/\s+',l): lines.append(tuple(chain))
rows=list(csv.reader(open(csvf))); hdr=rows[1]; data=rows[2:]
print(len(lines),len(data))
ix={h:i for i,h in enumerate(hdr)}
stalls=[h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
def phase(ch):
    st=[c[1] for c in ch if c[0]=='step_tile.cuh']
    if not st: return 'other'
    if any(903<=x<=970 for x in st): return 'stage_tile'
    inner=[x for x in st if 246<=x<=570]
    post=[x for x in st if 122<=x<=205]
    outer=st[-1]
    if post: return 'C.post'
    if inner:
        ln=inner[-1]
        tag = 'A' if ln<317 else ('B' if ln<424 else ('C.next' if 520<=ln<=557 else 'C'))
        return '%s@%d'%(tag,outer)
    return 'k@%d'%outer
agg=collections.defaultdict(collections.Counter); tot=collections.Counter()
for ch,r in zip(lines,data):
    p=phase(ch) if ch else 'none'
    a=agg[p]; ie=int(r[ix['Instructions Executed']]); sp=int(r[ix['# Samples']])
    a['inst']+=ie; a['samples']+=sp; tot['inst']+=ie; tot['samples']+=sp
    for s in stalls: a[s]+=int(r[ix[s]])
print('total inst',tot['inst'],'samples',tot['samples'])
for p,a in sorted(agg.items(), key=lambda x:-x[1]['inst']):
    if a['inst']/tot['inst']<0.002 and a['samples']/tot['samples']<0.003: continue
    top=sorted(((a[s],s[6:]) for s in stalls),reverse=True)[:4]
    print('%-14s %10d %6.2f%% %6.2f%% | %s'%(p,a['inst'],100*a['inst']/tot['inst'],100*a['samples']/tot['samples'],' '.join('%s:%.1f%%'%(s,100*v/tot['samples']) for v,s in top)))
