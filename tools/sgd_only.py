import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
import bench
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
for rep in range(2):
    r = bench.sgd_section(dev, steps=8)
    print(json.dumps({"all": [round(x, 2) for x in r["sgd_step_ms_all"]], "tttp": r["tttp_residual_ms"]}), flush=True)
    torch.cuda.empty_cache()
