import re,sys,subprocess
from collections import Counter
f,k=sys.argv[1],sys.argv[2]
out=subprocess.run(["cuobjdump","-sass","-fun",k,f],capture_output=True,text=True).stdout
ins=[]
for l in out.splitlines():
    m=re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?)\s*;",l)
    if m: ins.append((int(m.group(1),16),m.group(2)))
best=None
for i,(a,t) in enumerate(ins):
    m=re.search(r"BRA(?:\.U)?\s+(?:!?U?P\w+,\s*)?0x([0-9a-f]+)",t)
    if m and int(m.group(1),16)<a:
        body=[x for x in ins if int(m.group(1),16)<=x[0]<=a]
        w=sum('IMAD.WIDE' in x[1] or 'IMAD.HI' in x[1] for x in body)
        if w>=int(sys.argv[3]) and (best is None or len(body)<len(best)): best=body
c=Counter(x[1].split()[0] if not x[1].startswith('@') else x[1].split()[1] for x in best)
print(len(best), sorted(c.items(), key=lambda x:-x[1])[:16])
