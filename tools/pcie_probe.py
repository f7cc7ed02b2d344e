"""Host<->device copy bandwidth from pinned memory on this box: one vs several streams per
direction, and both directions at once (what bench.py's e2e leg can get)."""
import torch


def bw(nbytes, fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return nbytes * reps / (s.elapsed_time(e) * 1e-3) / 1e9


def main():
    n = 1 << 28  # 256 MiB per buffer
    dev = torch.device("cuda:0")
    hs = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(4)]
    ds = [torch.empty(n, dtype=torch.uint8, device=dev) for _ in range(4)]
    ho = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(4)]
    streams = [torch.cuda.Stream(dev) for _ in range(8)]
    cur = torch.cuda.current_stream()

    def copies(direction, k):
        def f():
            for i in range(4):
                st = streams[(i % k) + (4 if direction == "d2h" else 0)]
                st.wait_stream(cur)
                with torch.cuda.stream(st):
                    if direction == "h2d":
                        ds[i].copy_(hs[i], non_blocking=True)
                    else:
                        ho[i].copy_(ds[i], non_blocking=True)
            for st in streams:
                cur.wait_stream(st)
        return f

    for k in (1, 2, 4):
        print(f"H2D {k} stream(s): {bw(4 * n, copies('h2d', k)):.1f} GB/s", flush=True)
        print(f"D2H {k} stream(s): {bw(4 * n, copies('d2h', k)):.1f} GB/s", flush=True)

        def both():
            copies("h2d", k)()
            copies("d2h", k)()
        # issue both directions before waiting: overlapped
        def both_overlap():
            for i in range(4):
                for direction, off in (("h2d", 0), ("d2h", 4)):
                    st = streams[(i % k) + off]
                    st.wait_stream(cur)
                    with torch.cuda.stream(st):
                        if direction == "h2d":
                            ds[i].copy_(hs[i], non_blocking=True)
                        else:
                            ho[i].copy_(ds[i], non_blocking=True)
            for st in streams:
                cur.wait_stream(st)
        print(f"H2D+D2H overlapped, {k} stream(s) each: {bw(8 * n, both_overlap):.1f} GB/s total", flush=True)


if __name__ == "__main__":
    main()
