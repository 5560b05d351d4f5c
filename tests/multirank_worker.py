"""One rank of the 2-GPU sequence-sharded check (tests/test_gpu_multirank.py).

Launched by torch.distributed.run with one process per GPU.  Every rank draws
the same seeded K/V/q (so rank 0 can also build the whole cache), keeps its
contiguous token slice of each stream in its own cache, and calls the native
oq_attention_decode_sharded (fused K3 -> this rank's partial -> ONE
ncclAllGather -> rank-ordered merge), then the same step fused over peer
memory (P2PExchange / oq_attention_decode_p2p).  Rank 0 compares the output with the
single-GPU attention_decode over the whole cache and writes the result to the
file named by argv[1]."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    import paper_2605_21226_b200 as oq

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", world_size=world, rank=rank)
    B, Hq, Hkv, T = 2, 14, 2, 8192
    bd, bn = oq.default_bit_split(2)
    ek = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn, rotation_seed=41))
    ev = oq.Encoder(oq.CodecConfig(b_dir=bd, b_nrm=bn, rotation_seed=42))
    g = torch.Generator(device=dev).manual_seed(5)
    k = torch.randn((B * Hkv, T, 128), device=dev, generator=g)
    v = torch.randn((B * Hkv, T, 128), device=dev, generator=g)
    q = torch.randn((B, Hq, 128), device=dev, generator=g)
    kr = ek.compress(k.reshape(-1, 128)).reshape(B * Hkv, T, -1)
    vr = ev.compress(v.reshape(-1, 128)).reshape(B * Hkv, T, -1)
    per = T // world
    mine = oq.KVCache(ek, ev, B, Hkv, per)
    mine.pack(kr[:, rank * per:(rank + 1) * per].contiguous(),
              vr[:, rank * per:(rank + 1) * per].contiguous(), per)
    uid = [oq.NcclComm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = oq.NcclComm(world, uid[0], rank)
    info = comm.info()
    got = oq.attention_decode_sharded(q, mine, 0, per, comm)
    torch.cuda.synchronize()
    outs = [torch.empty_like(got) for _ in range(world)]
    dist.all_gather_object(outs, got.cpu())
    comm.close()
    # the same step fused over peer memory (CUDA IPC exchange buffers), twice
    xchg = oq.P2PExchange(mine, Hq)
    p2p = [xchg.decode(q, mine, 0, per) for _ in range(2)]
    torch.cuda.synchronize()
    p2p_outs = [None] * world
    dist.all_gather_object(p2p_outs, p2p[1].cpu())
    xchg.close()
    if rank == 0:
        full = oq.KVCache(ek, ev, B, Hkv, T)
        full.pack(kr, vr, T)
        want = oq.attention_decode(q, full).cpu()
        err = ((outs[0] - want).norm(dim=-1) / want.norm(dim=-1)).max().item()
        same = all(torch.equal(o, outs[0]) for o in outs)
        p2p_err = ((p2p_outs[0] - want).norm(dim=-1) / want.norm(dim=-1)).max().item()
        p2p_same = all(torch.equal(o, p2p_outs[0]) for o in p2p_outs)
        with open(sys.argv[1], "w") as f:
            json.dump({"nranks": info[1], "max_rel_err": err, "identical_on_ranks": same,
                       "p2p_max_rel_err": p2p_err, "p2p_identical_on_ranks": p2p_same}, f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
