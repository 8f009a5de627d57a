import os,sys
sys.path.insert(0,'/root/repo')
os.environ["CUTBDDC_SWEEP_STATS"]="1"
from paper_1703_06323_b200 import configs, cutbddc as cb
for name in sys.argv[1:]:
    cfg=configs.get(name); s=cb.GpuSolver(0); pb=cb.prepare(s,cfg)
    print("=====",name, file=sys.stderr, flush=True)
    s.setup_bddc(pb.objects,cfg.weighting); s.close()
