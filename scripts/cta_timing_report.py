"""Per-CTA phase report of K3 from scripts/cta_timing.py output:
python scripts/cta_timing_report.py <ts.npy> <number of CTAs of the launch>"""
import numpy as np, sys
n=int(sys.argv[2])
a=np.load(sys.argv[1])[:n].astype(np.int64)
t0=a[:,0]; base=t0.min()
t0=t0-base; t1=a[:,1]-base; t2=a[:,2]-base; t3=a[:,3]-base; t4=a[:,4]-base
sm=a[:,5]>>32; c=a[:,5]&0xffffffff; rounds=a[:,6]>>32; staged=a[:,6]&0xffffffff
dur=t4-t0
print('kernel span us', (t4.max())/1e3, 'CTAs', n)
print('CTA dur us: mean %.2f med %.2f p90 %.2f max %.2f'%(dur.mean()/1e3, np.median(dur)/1e3, np.percentile(dur,90)/1e3, dur.max()/1e3))
t8=a[:,8]-base; t9=a[:,9]-base
ph=[('start->l0',t1-t0),('l0->list',t8-t1),('list->issued',t9-t8),('issued->staged',t2-t9),('staged->lastacc',t3-t2),('lastacc->end',t4-t3)]
for k,v in ph: print('  %-16s mean %.2f us'%(k, v.mean()/1e3))
# per channel
for ch in np.unique(c):
    m=c==ch
    print('ch',ch,'n',m.sum(),'dur mean %.2f us'%(dur[m].mean()/1e3),'rounds mean %.2f'%rounds[m].mean(),'staged mean %.1f'%staged[m].mean(),
          ' phases', ' '.join('%.2f'%(v[m].mean()/1e3) for k,v in ph))
# concurrency: CTAs per SM over time
smn=sm.max()+1
print('SMs', smn, 'CTAs/SM', n/smn)
# total busy time per SM / span
busy=np.bincount(sm, weights=dur, minlength=smn)
print('per-SM sum dur / span: mean %.2f min %.2f max %.2f (resident CTAs avg)'%((busy/t4.max()).mean(), (busy/t4.max()).min(), (busy/t4.max()).max()))
# rounds dist
print('rounds hist', np.bincount(rounds)[:12])
