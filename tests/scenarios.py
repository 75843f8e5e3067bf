"""The reference's handcrafted-placement scenarios (proj/tests/test_table.cpp:41-206, test_bucket.cpp:25-77),
restated once and run against any table through a small adapter: the CPU oracle, the compiled reference, and the
CUDA path one key per launch (serial insertion makes slot positions exact on the GPU too)."""
import numpy as np

EMPTY = 0xFFFFFFFF


def pack(k, v):
    return (v << 32) | k


class OracleAdapter:
    """oracle.binding.OracleTable / RefTable."""

    def __init__(self, lib, cfg):
        self.t = lib.table(cfg)
        self.cfg = cfg

    def insert(self, k, v, prose=False):
        r, p = self.t.insert_pair(k, v, prose)
        return r == 1, p

    def find(self, k):
        found, v, p = self.t.find_key(k)
        return (v if found else None), p

    def locate(self, k):
        return self.t.locate(k)

    def poke(self, i, slot):
        self.t.poke_slot(i, slot)

    def inserted(self):
        return self.t.inserted

    def occupied(self):
        return self.t.occupied_slots()


class GpuAdapter:
    """paper_2108_07232_b200.HashTable, one key per bulk call."""

    def __init__(self, bht, cfg):
        self.bht = bht
        self.t = bht.HashTable(cfg, 0)

    def insert(self, k, v, prose=False):
        if self.t.kind == "iht":
            self.t.set_iht_prose_fallback(prose)
        o = self.t.insert(np.array([k], dtype=np.uint32), np.array([v], dtype=np.uint32))
        return o.success, o.probes

    def find(self, k):
        out, st = self.t.find(np.array([k], dtype=np.uint32), want_stats=True)
        return (None if out[0] == EMPTY else int(out[0])), st.probes

    def locate(self, k):
        st = self.t.download_store()
        idx = np.nonzero((st & np.uint64(0xFFFFFFFF)) == np.uint64(k))[0]
        return int(idx[0]) if idx.size else -1

    def poke(self, i, slot):
        self.t.poke_slot(i, slot)

    def inserted(self):
        return self.t.inserted()

    def occupied(self):
        return self.t.occupied_slots()


def scenario_bcht_empty_insert(make, make_config):
    # test_table.cpp:41-55
    t = make(make_config("bcht", 100, 0.5, 16, None, 3))
    assert t.insert(7, 42) == (True, 1)
    assert t.inserted() == 1
    assert t.find(7) == (42, 1)
    assert t.find(8)[0] is None


def scenario_cuckoo_cycle(make, craft):
    # test_table.cpp:57-73: a 2-cycle fails after max_chain exchanges = max_chain + 1 probes
    cfg = craft("1cht", 2, 1, [(1, 0, 2), (1, 1, 2), (1, 0, 2), (1, 1, 2)], 0, 8)
    t = make(cfg)
    assert t.insert(0, 1)[0]
    assert t.insert(2, 3)[0]
    ok, probes = t.insert(4, 5)
    assert not ok and probes == cfg.max_chain + 1
    assert t.occupied() == 2


def scenario_bp2ht_placement(make, craft):
    # test_table.cpp:85-103
    t = make(craft("bp2ht", 4, 2, [(1, 0, 4), (1, 1, 4)]))
    assert t.insert(0, 1) == (True, 2)   # buckets 0 and 1, tie -> bucket 0
    assert t.locate(0) == 0
    assert t.insert(4, 1) == (True, 2)   # bucket0 load 1, bucket1 load 0 -> bucket 1
    assert t.locate(4) == 2
    assert t.find(0) == (1, 1)           # hit in the first bucket
    assert t.find(8) == (None, 2)        # negative find always reads both


def scenario_bp2ht_both_full(make, craft):
    # test_table.cpp:105-114
    t = make(craft("bp2ht", 2, 1, [(1, 0, 2), (1, 1, 2)]))
    assert t.insert(0, 1)[0] and t.insert(2, 1)[0]
    assert not t.insert(4, 1)[0]
    assert t.occupied() == 2


def scenario_iht_threshold(make, craft):
    # test_table.cpp:125-146: `load >= t` sends the key to the secondaries
    t = make(craft("iht", 4, 2, [(1, 0, 4), (1, 1, 4), (1, 2, 4)], 2))
    assert t.insert(0, 1) == (True, 1)
    assert t.insert(4, 1) == (True, 1)
    assert t.insert(8, 1) == (True, 3)   # primary full: reads both secondaries
    assert t.locate(8) == 2              # secondary s0 = bucket 1
    assert t.find(0) == (1, 1)
    assert t.find(8) == (1, 2)           # miss primary, hit first secondary
    assert t.find(16) == (None, 3)       # negative find reads all three


def scenario_iht_fallback(make, craft):
    # test_table.cpp:148-190
    cfg = craft("iht", 4, 2, [(1, 0, 4), (1, 1, 4), (1, 2, 4)], 1)
    t = make(cfg)
    assert t.insert(1, 1)[0]
    assert t.locate(1) == 2
    t.poke(3, pack(0x999, 1))            # bucket 1 full
    assert t.insert(4, 1)[0]
    assert t.locate(4) == 0
    assert t.insert(8, 1)[0]             # s0 full, s1 empty -> s1
    assert t.locate(8) == 4
    t.poke(5, pack(0x998, 1))            # s1 full as well
    assert t.insert(12, 1)[0]            # both secondaries full -> back to the primary
    assert t.locate(12) == 1
    assert not t.insert(16, 1)[0]        # all three full
    p = make(cfg)
    p.poke(2, pack(0x999, 1)); p.poke(3, pack(0x999, 1)); p.poke(4, pack(0x998, 1)); p.poke(5, pack(0x998, 1))
    assert p.insert(4, 1)[0]                      # below threshold: primary
    assert not p.insert(8, 1, prose=True)[0]      # prose mode: both secondaries full is a failure
    assert p.insert(8, 1, prose=False)[0]         # listing fallback uses the primary


def scenario_bucket_ops(make, craft):
    # test_bucket.cpp:25-77 through the table: CAS lands on index = load, only on an empty slot; find takes the
    # lowest matching slot
    t = make(craft("bcht", 1, 16, [(1, 0, 1), (1, 0, 1), (1, 0, 1)], 0, 4))
    for i in range(16):
        ok, probes = t.insert(100 + i, i)
        assert ok and probes == 1
        assert t.locate(100 + i) == i    # slots fill in order
    assert t.occupied() == 16
    assert t.find(103) == (3, 1)
    t.poke(9, pack(103, 77))             # duplicate key further right: the lowest slot still wins
    assert t.find(103) == (3, 1)
    ok, probes = t.insert(500, 1)        # full single bucket, all hashes agree: evicts max_chain times then fails
    assert not ok and probes == 5
    assert t.occupied() == 16


ALL = [
    (scenario_bcht_empty_insert, "make_config"),
    (scenario_cuckoo_cycle, "craft"),
    (scenario_bp2ht_placement, "craft"),
    (scenario_bp2ht_both_full, "craft"),
    (scenario_iht_threshold, "craft"),
    (scenario_iht_fallback, "craft"),
    (scenario_bucket_ops, "craft"),
]
