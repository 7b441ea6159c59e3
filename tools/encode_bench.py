"""GPU encoder throughput (izg_encode; secondary path): C5-like
ClusterData arrays, device-resident values, CUDA events around the launch,
median of 10 after 3 warm-ups.  Verified: the words of every chunk equal the
harness host encoder's (itself word-for-word with the reference encoder,
tests/test_config_words.py), and the GPU decode of them returns the input.
Bytes moved = 4 per value read + 4 per payload word written."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import harness as H
import paper_1209_2137_b200 as P
from paper_1209_2137_b200 import _native as N

count = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
vals, _ = H.gen_arrays("cluster", count, 65536, (20, 29), seed=1)
flat = vals.reshape(-1)
offs = np.arange(count, dtype=np.uint64) * 65536
counts = np.full(count, 65536, np.uint32)
L = N.lib()
dv = torch.from_numpy(flat.view(np.int32)).cuda()
for name in ("simdbp128-s4", "simdfastpfor-s4"):
    codec = P.make_codec(name)
    bound = (int(L.izg_encode_bound(codec.codec, 65536)) + 3) // 4 * 4
    table = np.zeros(count, dtype=N.CHUNK_DTYPE)
    table["word_off"] = np.arange(count, dtype=np.uint64) * bound
    table["n"] = counts
    table["out_off"] = offs
    d_table0 = torch.from_numpy(table.view(np.uint8)).cuda()
    d_table = d_table0.clone()
    d_words = torch.zeros(count * bound + 4, dtype=torch.int32, device="cuda")
    d_status = torch.full((count,), -1, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    def run():
        d_table.copy_(d_table0)
        rc = L.izg_encode(codec.codec, codec.delta, N.ptr(dv), N.ptr(d_table), count, N.ptr(d_words),
                          N.ptr(d_status), 0, s.cuda_stream)
        assert rc == N.SUCCESS, rc
    ts = []
    for i in range(13):
        d_table.copy_(d_table0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rc = L.izg_encode(codec.codec, codec.delta, N.ptr(dv), N.ptr(d_table), count, N.ptr(d_words),
                          N.ptr(d_status), 0, s.cuda_stream)
        e1.record(); torch.cuda.synchronize()
        assert rc == N.SUCCESS, rc
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    assert (d_status.cpu().numpy() == 0).all()
    t = float(np.median(ts)) * 1e-3
    out_table = d_table.cpu().numpy().view(N.CHUNK_DTYPE)
    words = d_words.cpu().numpy().view(np.uint32)
    ref = H.encode_chunks(codec, flat, offs, counts)
    same = True
    for i in range(count):
        a = words[int(out_table["word_off"][i]):int(out_table["word_off"][i]) + int(out_table["n_words"][i])]
        b = ref.words[int(ref.table["word_off"][i]):int(ref.table["word_off"][i]) + int(ref.table["n_words"][i])]
        if len(a) != len(b) or not np.array_equal(a, b):
            same = False
            break
    nw = int(out_table["n_words"].sum())
    print(json.dumps({"codec": name, "arrays": count, "ms": round(t * 1e3, 4),
                      "G_int_per_s": round(flat.size / t / 1e9, 1),
                      "GBps": round((4 * flat.size + 4 * nw) / t / 1e9, 1),
                      "bits_per_int": round(32 * nw / flat.size, 3),
                      "words_equal_host_encoder": bool(same)}), flush=True)
