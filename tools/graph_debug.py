#!/usr/bin/env python
"""Debug aid: capture one pipeline step into a CUDA graph call by call and report which ABI call
fails under capture (and with which capture mode)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_2407_16990_b200 as rg  # noqa: E402


def main():
    wl = synth.CONFIGS["c2"]
    imp = torch.from_numpy(synth.importance_maps(wl.S, wl.F, wl.GH, wl.GW, 0, "blobs")).cuda()
    fr = torch.from_numpy(synth.frames_rgb8(wl.S, wl.F, wl.H, wl.W, 0)).cuda()
    w = synth.sr_weights(wl.sr, 0)
    p = rg.Pipeline(S=wl.S, F=wl.F, W=wl.W, H=wl.H, k=wl.k, bin_w=wl.bin_w, bin_h=wl.bin_h, max_bins=wl.max_bins,
                    partition_mb=wl.partition_mb, scale=wl.sr.scale, channels=wl.sr.channels,
                    n_resblocks=wl.sr.n_resblocks, weights=w, bf16=wl.sr.bf16)
    for _ in range(2):
        p.run(imp, fr)
    torch.cuda.synchronize()
    for mode in ("global", "thread_local", "relaxed"):
        for name, fn in (("select", lambda s: p.select(imp, stream=s)), ("pack", lambda s: p.pack_step(imp, stream=s)),
                         ("enhance_scatter", lambda s: p.enhance_scatter(fr, stream=s))):
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            try:
                with torch.cuda.graph(g, stream=s, capture_error_mode=mode):
                    fn(s)
                g.replay()
                torch.cuda.synchronize()
                print(mode, name, "OK")
            except Exception as e:  # noqa: BLE001
                print(mode, name, "FAIL", str(e)[:300])
                torch.cuda.synchronize()
    # the bench structure: capture stream + two worker streams joined by events
    cap, s1, s2 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    e1, e2 = torch.cuda.Event(), torch.cuda.Event()
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g, stream=cap):
            s1.wait_stream(cap)
            s2.wait_stream(cap)
            with torch.cuda.stream(s1):
                print("in capture: s1 status", s1.query() if False else "-", flush=True)
                p.select(imp, stream=s1)
                p.pack_step(imp, stream=s1)
                e1.record(s1)
            with torch.cuda.stream(s2):
                s2.wait_event(e1)
                p.enhance_scatter(fr, stream=s2)
                e2.record(s2)
            cap.wait_stream(s1)
            cap.wait_stream(s2)
        g.replay()
        torch.cuda.synchronize()
        print("cross-stream OK")
    except Exception as e:  # noqa: BLE001
        print("cross-stream FAIL", str(e)[:400])
    # exactly the bench schedule: two pipelines, events, warm pipelined steps, then capture
    pipes = [p, rg.Pipeline(S=wl.S, F=wl.F, W=wl.W, H=wl.H, k=wl.k, bin_w=wl.bin_w, bin_h=wl.bin_h,
                            max_bins=wl.max_bins, partition_mb=wl.partition_mb, scale=wl.sr.scale,
                            channels=wl.sr.channels, n_resblocks=wl.sr.n_resblocks, weights=w, bf16=wl.sr.bf16)]
    s_front, s_back = torch.cuda.Stream(), torch.cuda.Stream()
    front_done = [torch.cuda.Event() for _ in range(2)]
    back_done = [torch.cuda.Event() for _ in range(2)]

    def steps(n, capturing=False):
        for k in range(n):
            q = pipes[k % 2]
            with torch.cuda.stream(s_front):
                if not (capturing and k < 2):
                    s_front.wait_event(back_done[k % 2])
                q.select(imp, stream=s_front)
                q.pack_step(imp, stream=s_front)
                front_done[k % 2].record(s_front)
            with torch.cuda.stream(s_back):
                s_back.wait_event(front_done[k % 2])
                q.enhance_scatter(fr, stream=s_back)
                back_done[k % 2].record(s_back)

    steps(3)
    torch.cuda.synchronize()
    for variant in range(2):
        cap = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        try:
            with torch.cuda.graph(g, stream=cap):
                s_front.wait_stream(cap)
                s_back.wait_stream(cap)
                steps(3, capturing=True)
                cap.wait_stream(s_front)
                cap.wait_stream(s_back)
            g.replay()
            torch.cuda.synchronize()
            print("bench schedule OK", variant)
        except Exception as e:  # noqa: BLE001
            import traceback
            traceback.print_exc()
            print("bench schedule FAIL", variant, str(e)[:400])
            torch.cuda.synchronize()
    # tracing inside a captured graph
    rg.trace_read()
    cap = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    rg.trace_enable(True)
    with torch.cuda.graph(g, stream=cap):
        s_front.wait_stream(cap)
        s_back.wait_stream(cap)
        steps(2, capturing=True)
        cap.wait_stream(s_front)
        cap.wait_stream(s_back)
    rg.trace_enable(False)
    g.replay()
    torch.cuda.synchronize()
    tr = rg.trace_read()
    print("traced in graph:", len(tr), tr[:6], tr[-4:])
    p.run(imp, fr)
    torch.cuda.synchronize()
    print("run after trace OK")


if __name__ == "__main__":
    main()
