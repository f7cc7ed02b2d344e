"""Page allocator of the paged KV cache: the host-side bookkeeping of PagedKVCache
(paged_kv.hpp:50-89, paged_kv.cpp:13-152). Pure host logic (no device work), so it is
shared by PagedKVCache and tested on CPU against the reference's page tables.

LIFO free list with page 0 popped first (paged_kv.cpp:27-31); deterministic_shuffle of the
free list (random.hpp:49-56); assign / append / erase with atomic capacity checks
(OutOfPages leaves the cache unchanged, paged_kv.cpp:81-87)."""
from __future__ import annotations

SENTINEL = -1
_M64 = (1 << 64) - 1


class OutOfPagesError(RuntimeError):
    pass


def _splitmix(state):
    state = (state + 0x9E3779B97F4A7C15) & _M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return state, z ^ (z >> 31)


class PageAllocator:
    def __init__(self, batches: int, num_pages: int, page_size: int):
        if batches < 1 or num_pages < 1 or page_size < 1:
            raise ValueError("PagedKVCache: batches, num_pages and page_size must be >= 1")
        self.batches, self.num_pages, self.ps = batches, num_pages, page_size
        self.table = [SENTINEL] * (batches * num_pages)
        self.phys_to_logical = [SENTINEL] * num_pages
        self.owner = [SENTINEL] * num_pages
        self.seq = [0] * batches
        self.free = [num_pages - 1 - p for p in range(num_pages)]  # LIFO: page 0 on top

    def shuffle_free_pages(self, seed: int):
        state = seed & _M64
        v = self.free
        for i in range(len(v), 1, -1):
            state, z = _splitmix(state)
            j = z % i
            v[i - 1], v[j] = v[j], v[i - 1]

    def check_batch(self, b):
        if b < 0 or b >= self.batches:
            raise IndexError(f"PagedKVCache: batch {b} outside [0, {self.batches})")

    def _take(self, b, lp):
        page = self.free.pop()
        self.table[b * self.num_pages + lp] = page
        self.phys_to_logical[page] = lp
        self.owner[page] = b

    def erase(self, b):
        self.check_batch(b)
        for lp in range(-(-self.seq[b] // self.ps)):
            slot = b * self.num_pages + lp
            page = self.table[slot]
            self.table[slot] = SENTINEL
            self.phys_to_logical[page] = SENTINEL
            self.owner[page] = SENTINEL
            self.free.append(page)
        self.seq[b] = 0

    def assign(self, b, n_tokens: int):
        """assign (paged_kv.cpp:72-98): returns the pages now backing batch b."""
        self.check_batch(b)
        needed = -(-n_tokens // self.ps)
        owned = -(-self.seq[b] // self.ps)
        if needed > len(self.free) + owned:
            raise OutOfPagesError(f"PagedKVCache: assign of {n_tokens} tokens needs {needed} pages, "
                                  f"only {len(self.free) + owned} available")
        self.erase(b)
        for lp in range(needed):
            self._take(b, lp)
        self.seq[b] = n_tokens

    def append(self, b, n_tokens: int):
        """append_tokens (paged_kv.cpp:100-126)."""
        self.check_batch(b)
        old = self.seq[b]
        owned, total = -(-old // self.ps), -(-(old + n_tokens) // self.ps)
        if total - owned > len(self.free):
            raise OutOfPagesError(f"PagedKVCache: append of {n_tokens} tokens needs {total - owned} new "
                                  f"pages, only {len(self.free)} free")
        for lp in range(owned, total):
            self._take(b, lp)
        self.seq[b] = old + n_tokens

    def lookup(self, b, logical_page):
        return self.table[b * self.num_pages + logical_page]
