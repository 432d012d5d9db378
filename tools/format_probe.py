import sys; sys.path.insert(0,'/root/repo')
import paper_2304_08232_b200 as slab
c=slab.Context(0); c.set_process_grid((2,1,1),0)
h=c.build_hierarchy((104,104,104),4)
l=h
while l is not None:
    print(l.n(), l.format_info(), l.A.format_info()); l=l.coarser
