"""Oracle restatement of the rule-group executor (``sparsewire/updates.py``).

Only what the hot path needs: rule ids in registration order
(updates.py:300-302), per-binding update counters (:366), host stream
(seed,"host",rule_id,update,pass) (:346-349), per-row child streams of
(seed,"row",rule_id,update,pass) (:313-318), the pass loop and its runaway
cap (:361-365), and remap-if-changed (:367-372).  Test infrastructure only.
"""

from __future__ import annotations

from .rng import Stream, fold_key, child_key


class Binding:
    def __init__(self, rule, rule_id, matrix_name):
        self.rule = rule
        self.rule_id = rule_id
        self.matrix_name = matrix_name
        self.update_count = 0


class HostCtx:
    def __init__(self, rng, pass_index):
        self.rng = rng
        self.pass_index = pass_index


class OracleModel:
    def __init__(self, seed):
        self.seed = seed
        self.matrices = {}
        self.groups = {}
        self.transposes = {}     # matrix name -> callable rebuild()
        self.next_rule_id = 0

    def add_matrix(self, name, m):
        self.matrices[name] = m

    def add_rule(self, group, matrix_name, rule):
        b = Binding(rule, self.next_rule_id, matrix_name)
        self.next_rule_id += 1
        self.groups.setdefault(group, []).append(b)
        return b

    def run_update_group(self, group):
        for b in self.groups[group]:
            rule = b.rule
            m = self.matrices[b.matrix_name]
            v0 = m.version
            p = 0
            while True:
                hctx = HostCtx(Stream.of(self.seed, "host", b.rule_id, b.update_count, p), p)
                rule.host_phase(hctx)
                rows = rule.active_rows(hctx)
                base = fold_key(self.seed, "row", b.rule_id, b.update_count, p)
                for r in rows:
                    rule.row_phase(int(r), Stream(child_key(base, int(r))))
                p += 1
                if not rule.continue_after_pass(hctx):
                    break
                if p > 2 * m.num_pre + 16:
                    raise RuntimeError("did not converge")
            b.update_count += 1
            tm = self.transposes.get(b.matrix_name)
            if tm is not None and m.version != v0:
                tm()
