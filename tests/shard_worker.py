"""One rank of a multi-process sharded run (test infrastructure, launched by
tests/test_gpu_shard_mp.py): the consolidation recipe from the reference's
builder, this rank's shard, ShardedEngine with the exchange backend given
(gloo: host-staged allgather, several ranks may share one GPU), the global
spike list and this rank's cell states written to an .npz."""
import os
import sys

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle")]
import numpy as np
import torch
import torch.distributed as dist

import ref
from paper_2411_16445_b200 import EngineOptions, shard


def main(out, n_cells, t_end, backend):
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dist.init_process_group(backend, rank=rank, world_size=world)
    cfg = ref.default_consolidation(n_cells=n_cells, n_exc=n_cells * 4 // 5, pattern=n_cells // 8,
                                    t_learn_ms=300.0, dt_ms=0.5, seed=5, multi_compartment=1)
    rr = ref.RefRecipe.consolidation(cfg)
    sh = shard.ShardedEngine(rr.view, EngineOptions(0.5, 5), rank, world, device=0,
                             record_spikes=True, backend=backend)
    for t in (200.0, t_end):
        sh.advance_to(t)
    t, g = sh.spike_arrays()
    b, e = sh.engine.gid_range()
    v = np.concatenate([sh.engine.cell(x).v_mV for x in range(b, e)])
    h = np.concatenate([sh.engine.cell(x).groups[0].stc_h for x in range(b, min(e, cfg.n_exc))] or [np.zeros(0)])
    np.savez(out, t=t, g=g, v=v, h=h, b=b, e=e)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), float(sys.argv[3]), sys.argv[4])
