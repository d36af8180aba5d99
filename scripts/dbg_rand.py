"""Debug the randomized segment test: print configs whose records differ."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import test_gpu_segments as T  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 2
captured = {}
orig = T._serial_and_segmented


def capture(pset, wl, ca, **env):
    captured.update(pset=pset, wl=wl, ca=ca, env=env)
    raise SystemExit(0)


T._serial_and_segmented = capture
try:
    T.test_segmented_random_sweeps_equal_serial(seed)
except SystemExit:
    pass
pset, wl, ca, env = captured["pset"], captured["wl"], captured["ca"], captured["env"]
print("env", env)
ser, _ = T._run(pset, wl, ca, {"TWB_SIM_SEG": "0"})
seg, _ = T._run(pset, wl, ca, {k: str(v) for k, v in env.items()})
bad = [c for c in range(len(ca)) if any(ser.results[f][c] != seg.results[f][c] for f in T.FIELDS)]
print("bad configs", len(bad), bad[:20])
for c in bad[:6]:
    cf = ca[c]
    print(c, {k: int(cf[k]) for k in ("chunk_size", "max_batch_tokens", "max_running", "kv_capacity_blocks", "pp_stages",
                                      "workers_per_replica", "policy", "pred_id", "workload_id", "tk_cooldown_ns", "flags", "epoch_ns")},
          "n", int(wl.wl_off[cf["workload_id"] + 1] - wl.wl_off[cf["workload_id"]]))
    for f in ("status", "steps", "tk_seq", "tk_offset_ns", "tk_wall_ns", "final_now_ns"):
        print("   ", f, int(ser.results[f][c]), int(seg.results[f][c]))
# isolate: run the first bad config alone, segmented, with stats
import torch  # noqa: E402
from paper_2601_00397_b200 import _lib  # noqa: E402
from paper_2601_00397_b200.sweep import DeviceSweep  # noqa: E402
if bad:
    c = bad[0]
    one = ca[c:c + 1].copy()
    for W in (1, 2, 4, 8, 16, 64):
        os.environ["TWB_SIM_SEG_W"] = str(W)
        os.environ["TWB_SIM_SEG_CAPDIV"] = str(env.get("TWB_SIM_SEG_CAPDIV", 1))
        d = DeviceSweep(pset, wl, one, per_request=True)
        st = torch.zeros(8, dtype=torch.int32, device="cuda")
        _lib.load().tw_sim_set_seg_stats(st.data_ptr())
        d.run()
        torch.cuda.synchronize()
        _lib.load().tw_sim_set_seg_stats(None)
        r = d.fetch().results[0]
        print("alone W", W, "offset", int(r["tk_offset_ns"]), "seq", int(r["tk_seq"]), "wall", int(r["tk_wall_ns"]),
              "stats", st.cpu().numpy().tolist())

# the bad config alone at the sweep's W, with the segment summaries decoded from scratch
if bad:
    c = bad[0]
    one = ca[c:c + 1].copy()
    os.environ["TWB_SIM_SEG_W"] = str(env["TWB_SIM_SEG_W"])
    os.environ["TWB_SIM_SEG_CAPDIV"] = os.environ.get("DBG_CAPDIV", str(env["TWB_SIM_SEG_CAPDIV"]))
    d = DeviceSweep(pset, wl, one, per_request=True)
    st = torch.zeros(8, dtype=torch.int32, device="cuda")
    _lib.load().tw_sim_set_seg_stats(st.data_ptr())
    d.run()
    torch.cuda.synchronize()
    _lib.load().tw_sim_set_seg_stats(None)
    r = d.fetch().results[0]
    print("alone W", env["TWB_SIM_SEG_W"], "offset", int(r["tk_offset_ns"]), "wall", int(r["tk_wall_ns"]), "stats", st.cpu().numpy().tolist())
    raw = d.d_scratch.cpu().numpy()
    W = int(raw[64:68].view(np.int32)[0])
    a256 = lambda x: (x + 255) & ~255
    wmax = env["TWB_SIM_SEG_W"]
    o = 64 + a256(4 * 1)
    a0s = raw[o:o + 4 * wmax].view(np.int32)
    o += a256(4 * wmax)
    SS = np.dtype([("j_stop", "<i4"), ("status", "<i4"), ("last_regen", "<i4"), ("adm_end", "<i4"), ("final_now", "<i8"),
                   ("events", "<i8"), ("dig", "<u8"), ("msum", "<u8"), ("steps", "<i4"), ("pred_code", "<i4"),
                   ("log_len", "<i4"), ("pad", "<i4"), ("wall", "<i8"), ("seq", "<i8"), ("lb", "<i8"), ("off", "<i8"),
                   ("disp", "<i4"), ("pad2", "<i4"), ("d_lo", "<i8"), ("d_hi", "<i8")])
    print("SegSummary itemsize", SS.itemsize)
    summ = raw[o:o + SS.itemsize * wmax].view(SS)
    print("W", W, "a0s", a0s.tolist())
    for w in range(W):
        print(w, {k: int(summ[w][k]) for k in ("j_stop", "status", "last_regen", "adm_end", "log_len", "wall", "seq", "off", "disp")})

# the whole sweep again, decoding the bad config's segments from the sweep's scratch
if bad:
    os.environ["TWB_SIM_SEG_W"] = str(env["TWB_SIM_SEG_W"])
    os.environ["TWB_SIM_SEG_CAPDIV"] = str(env["TWB_SIM_SEG_CAPDIV"])
    d = DeviceSweep(pset, wl, ca, per_request=True)
    nc = len(ca)
    st = torch.zeros(8 * nc, dtype=torch.int32, device="cuda")
    _lib.load().tw_sim_set_seg_stats(st.data_ptr())
    d.run()
    torch.cuda.synchronize()
    _lib.load().tw_sim_set_seg_stats(None)
    res = d.fetch().results
    raw = d.d_scratch.cpu().numpy()
    wmax = env["TWB_SIM_SEG_W"]
    o = 64 + a256(4 * nc)
    nseg = raw[64:64 + 4 * nc].view(np.int32)
    a0all = raw[o:o + 4 * nc * wmax].view(np.int32).reshape(nc, wmax)
    o += a256(4 * nc * wmax)
    summ = raw[o:o + SS.itemsize * nc * wmax].view(SS).reshape(nc, wmax)
    for c in bad[:2]:
        print("sweep config", c, "offset", int(res["tk_offset_ns"][c]), "wall", int(res["tk_wall_ns"][c]),
              "stats", st.view(-1, 8)[c].cpu().numpy().tolist(), "W", int(nseg[c]), "a0s", a0all[c].tolist())
        for w in range(int(nseg[c])):
            print("  ", w, {k: int(summ[c, w][k]) for k in ("j_stop", "status", "last_regen", "adm_end", "log_len", "wall", "seq", "off", "disp", "d_lo", "d_hi")})

if bad:
    c = bad[0]
    S = raw.size
    hdr = a256(64 + a256(4 * nc) + a256(4 * nc * wmax) + a256(SS.itemsize * nc * wmax))
    xtra = max(64, min(4096, (256 << 20) // ((8 * 24 + 64) * nc * wmax)))
    fixed = hdr + xtra * nc * wmax * 256
    r_max = (S - fixed - 1024) // 332
    regpos = raw[hdr:hdr + 4 * r_max].view(np.int32)
    RG = np.dtype([("events", "<i8"), ("dig", "<u8"), ("msum", "<u8"), ("steps", "<i4"), ("pad", "<i4"),
                   ("wall", "<i8"), ("seq", "<i8"), ("lb", "<i8"), ("off", "<i8"), ("disp", "<i4"), ("pad2", "<i4")])
    ro = hdr + a256(4 * r_max)
    reg = raw[ro:ro + RG.itemsize * r_max].view(RG)
    rb = int(d.req_base[c])
    print("xtra", xtra, "r_max", r_max, "rb", rb)
    for j in list(range(0, 15)) + list(range(105, 125)) + list(range(225, 240)):
        if regpos[rb + j] >= 0:
            print("  regen", j, "pos", int(regpos[rb + j]), {k: int(reg[rb + j][k]) for k in ("events", "steps", "wall", "seq", "lb", "off", "disp")})
