import sys; sys.path.insert(0,'.')
from paper_2207_00032_b200 import engine as E
for B in (1,16):
  for (N,K) in [(12288,4096),(4096,4096),(16384,4096),(4096,16384),(50304,4096)]:
    for i8 in (False,True):
      p=E.launch_plan(N,K,B,i8); print(B,N,K,"i8" if i8 else "f16", "split",p.ksplit,"rps",p.rows_per_split,"ctas",p.ctas,"stages",p.stages)
