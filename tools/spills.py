import re,sys
cur=None
for l in open(sys.argv[1]):
    m=re.search(r"Compiling entry function '(\S+)'",l)
    if m:
        n=m.group(1)
        mm=re.search(r'kernelILi(\d+)ENS_6MaskFnILi(\d)EEENS_7ScoreFnILi(\d)',n)
        cur=('D=%s M=%s S=%s'%mm.groups()) if mm else n[:70]
        continue
    if 'spill' in l and cur:
        print(cur, l.strip().replace('ptxas info    : ','')); cur=None
    m=re.search(r'Used (\d+) registers',l)
