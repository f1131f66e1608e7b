# Needs a probe build: make -C paper_2510_06710_b200/csrc EXTRA=-DCKRL_PROBES (or CKRL_LIB=<such a build>).
import sys, os, ctypes as C, torch
sys.path.insert(0, os.getcwd())
import paper_2510_06710_b200 as ck
from paper_2510_06710_b200 import optim, synth, _lib
from paper_2510_06710_b200.core import *
name = sys.argv[1] if len(sys.argv) > 1 else 'cfg3'
cfg = synth.CONFIGS[name]; a,l,v = synth.SPECS[name]
d = synth.episodes_numpy(cfg); lg, tk, old = synth.token_tensors(cfg)
d['tokens'], d['old_logprob'] = tk, old
ro = RolloutBuffer.from_arrays(d, d['boot_scalar'] if a == 0 else d['boot_vector0'], 256)
pol = PolicyOutputs(lg, torch.tensor(d['new_value_scalar'] if v == 0 else d['new_value_vector'], dtype=torch.float32, device='cuda'))
st = optim.PpoStep(ro, GaeParams(), GranularitySpec(Level(a), Level(l), Level(v)), PpoParams(0.2, 0.5, 0.01, True))
for i in range(5): st(ro, pol)
torch.cuda.synchronize()
buf = (C.c_uint64 * 32)()
_lib.check(_lib.lib().ckrl_debug_timeline(buf, 32))
t0 = buf[0]
names = {0:'start',1:'u0store',2:'u0issue',3:'u1rowfull',28:'u1store',29:'u1issue',30:'u1done',31:'u1tokpass',1:'gaeA',2:'gridbar',3:'consts',4:'unit0',8:'rowlast',9:'alldone',10:'reduced',11:'r0meta',12:'r0full',13:'r0done',14:'r1meta',15:'r1full',16:'r1done',17:'r2meta',18:'r2full',19:'r2done',20:'b0rowfull',24:'b0meta0',25:'red_sync',26:'red_fence',27:'red_ticket'}
print(name, ' '.join(f"{names[i]}={(buf[i]-t0)/1000:.2f}" for i in sorted(names) if buf[i] >= t0 and buf[i]-t0 < 10**9))


# kernel-level view: CUDA events around one step (assembly + loss), for comparison with the marks
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); st(ro, pol); e1.record(); torch.cuda.synchronize()
_lib.check(_lib.lib().ckrl_debug_timeline(buf, 32))
print('  step event us=%.2f  cta0 start->reduced us=%.2f' % (e0.elapsed_time(e1) * 1e3, (buf[10] - buf[0]) / 1000))
