"""Oracle restatement of the logits-cache index and slab allocator
(TEST INFRASTRUCTURE ONLY).

Semantics restated from ``pkg/src/agentserve/logits_cache.py``:

* ``lookup`` (logits_cache.py:87-94): ``lookups += 1``; on a hit the hit
  clock ticks, the entry's ``last_hit`` takes the new clock, ``hits += 1``.
  Misses do not tick.
* ``update`` (logits_cache.py:96-126): overwrite subtracts the old entry's
  accounted bytes and creates a *new* entry (pins reset); the clock ticks;
  the entry's ``last_hit`` takes the clock; accounted bytes
  ``n*V*4 + 8*n`` (logits_cache.py:54-56, TOKEN_OVERHEAD_BYTES :23) are
  added; then ``_evict_over_budget`` (logits_cache.py:128-140).
* eviction: while ``total > budget and len > 1`` evict the unpinned entry
  with minimal ``(last_hit, digest)``; the new entry itself is eligible; stop
  if every entry is pinned.
* ``pin`` / ``unpin`` (logits_cache.py:145-149) act on an entry *object*: a
  pin taken before an overwrite stays on the old object.  Here that object is
  the (slot, generation) pair.

What the reference does not define and this restatement fixes (the GPU
allocator must match it bit-for-bit -- "cache slot indices bit-exact"):

* entry slots come from a LIFO free stack, initially ``0, 1, 2, ...``;
  an overwrite keeps the key's slot and bumps its generation;
* row pages (``page_rows`` rows each) come from a LIFO free stack, initially
  ``0, 1, 2, ...``; at each insert the overwritten entry's pages are pushed
  first (in REVERSE page order, so the new entry gets them back in place),
  then the new entry's pages are popped, then each victim's pages are pushed
  (in page order) as it is evicted;
* a batch of operations is the sequence of its elements in index order.
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass, field

TOKEN_OVERHEAD_BYTES = 8


@dataclass
class Entry:
    digest: int
    slot: int
    gen: int
    n: int
    vocab: int
    last_hit: int
    pages: list[int]
    pins: int = 0
    tokens: list[int] = field(default_factory=list)

    @property
    def nbytes(self) -> int:
        return self.n * self.vocab * 4 + TOKEN_OVERHEAD_BYTES * self.n


class CacheOracle:
    def __init__(self, budget_bytes: int, key_capacity: int, page_capacity: int, page_rows: int = 1,
                 heap: bool = False):
        """``heap=False`` finds each victim by the reference's linear scan for the
        minimal ``(last_hit, digest)`` (logits_cache.py:131-137); ``heap=True``
        keeps a lazy min-heap of ``(last_hit, digest)`` ticks instead -- the same
        victims (ticks are unique), O(log E) per eviction, for C4-sized traces."""
        self.budget = budget_bytes
        self.heap = [] if heap else None
        self.page_rows = page_rows
        self.entries: dict[int, Entry] = {}
        self.by_slot: dict[int, Entry] = {}
        self.gen = [0] * key_capacity
        self.free_slots = list(range(key_capacity - 1, -1, -1))  # pop() -> 0, 1, ...
        self.free_pages = list(range(page_capacity - 1, -1, -1))
        self.total = 0
        self.clock = 0
        self.lookups = 0
        self.hits = 0
        self.inserts = 0
        self.evictions = 0
        self.capacity_errors = 0

    def __len__(self):
        return len(self.entries)

    # lookup: logits_cache.py:87-94
    def lookup(self, digest: int):
        self.lookups += 1
        e = self.entries.get(digest)
        if e is None:
            return None
        self.clock += 1
        e.last_hit = self.clock
        self.hits += 1
        if self.heap is not None:
            heapq.heappush(self.heap, (self.clock, digest))
        return e

    def _pages_for(self, n: int) -> int:
        return -(-n // self.page_rows)

    # update: logits_cache.py:96-140
    def insert(self, digest: int, n: int, vocab: int, tokens=()):
        """Returns (entry, [evicted (digest, slot, gen)])."""
        old = self.entries.get(digest)
        if old is not None:
            self.total -= old.nbytes
            # pushed in reverse page order: the new entry's pops (page 0 first) return
            # them in place, so a write-back's replayed prefix rows need no copy
            for p in reversed(old.pages):
                self.free_pages.append(p)
            slot = old.slot
            self.gen[slot] += 1
        else:
            if not self.free_slots:
                raise MemoryError("entry slots exhausted")
            slot = self.free_slots.pop()
        npages = self._pages_for(n)
        if len(self.free_pages) < npages:
            # out of slab pages (the reference has no slab): the insert is rolled back -- the
            # key leaves the cache (an overwritten entry is already gone) and its slot returns
            # to the free stack; the GPU latches LC_E_CAPACITY
            if old is not None:
                del self.entries[digest]
                del self.by_slot[slot]
            self.free_slots.append(slot)
            self.capacity_errors += 1
            return None, []
        pages = [self.free_pages.pop() for _ in range(npages)]
        self.clock += 1
        e = Entry(digest, slot, self.gen[slot], n, vocab, self.clock, pages, 0, list(tokens))
        self.entries[digest] = e
        self.by_slot[slot] = e
        self.total += e.nbytes
        self.inserts += 1
        if self.heap is not None:
            heapq.heappush(self.heap, (self.clock, digest))
        victims = []
        held = []  # pinned heap items, pushed back after this insert
        while self.total > self.budget and len(self.entries) > 1:
            if self.heap is None:
                cands = [(v.last_hit, d) for d, v in self.entries.items() if v.pins == 0]
                if not cands:
                    break
                _, d = min(cands)
            else:
                d = None
                while self.heap:
                    ck, dd = heapq.heappop(self.heap)
                    v = self.entries.get(dd)
                    if v is None or v.last_hit != ck:
                        continue  # stale tick
                    if v.pins:
                        held.append((ck, dd))
                        continue
                    d = dd
                    break
                if d is None:
                    break
            v = self.entries.pop(d)
            del self.by_slot[v.slot]
            self.total -= v.nbytes
            for p in v.pages:
                self.free_pages.append(p)
            self.free_slots.append(v.slot)
            self.gen[v.slot] += 1
            self.evictions += 1
            victims.append((v.digest, v.slot, v.gen))
        for it in held:
            heapq.heappush(self.heap, it)
        return e, victims

    def pin(self, slot: int, gen: int, delta: int = 1):
        e = self.by_slot.get(slot)
        if e is not None and e.gen == gen:
            e.pins += delta

    def unpin(self, slot: int, gen: int):
        self.pin(slot, gen, -1)
