"""Oracle: operator-graph DSL parser, canonical printer and dependency validator.

Test infrastructure only (see oracle/__init__.py).  Independent re-implementation of
the rules the product's C++ validator enforces; the two must agree on accept/reject.

Sources
  * operators and stages: P:11-31 (draft §Operator), P:275-281 (§IV-A)
  * "operators prefixed with BMW and BMT cannot be followed by operators prefixed with
    BMTB": P:36 (draft), P:292 (§IV-B)
  * "COMPRESS, the last operator in converting stage" P:22; "mapping stage always begins
    after the COMPRESS operator" P:279
  * name aliases (draft vs final, typos): P:29 footnote, P:281, P:351 — reading A37
  * the full rule list R1-R11 is reading A16

Grammar (DESIGN.md §Graph DSL):
  seq := op (';' op)* ;  op := NAME ['(' [arg (',' arg)*] ')'] ['{' seq ('|' seq)* '}']
  arg := [KEY '='] value ;  value := NUMBER | '[' [NUMBER (',' NUMBER)*] ']' | IDENT
"""
from __future__ import annotations

import dataclasses
import re
from typing import Any

CONVERTING = {"ROW_DIV", "COL_DIV", "SORT", "SORT_SUB", "BIN", "DIA_DECOM", "DENSE_DECOM", "HYB_DECOM"}
MAPPING = {"BMTB_ROW_BLOCK", "BMTB_NNZ_BLOCK", "BMW_ROW_BLOCK", "BMW_NNZ_BLOCK",
           "BMT_ROW_BLOCK", "BMT_NNZ_BLOCK", "BMT_PAD", "SORT_BMTB"}
REDUCTIONS = {"THREAD_TOTAL_RED": "BMT", "THREAD_BITMAP_RED_G": "BMT",
              "WARP_TOTAL_RED": "BMW", "WARP_BITMAP_RED": "BMW", "WARP_SEG_ADD_RED": "BMW",
              "SHMEM_TOTAL_RED": "BMTB", "SHMEM_OFFSET_RED": "BMTB", "GMEM_ATOM_RED": "GMEM"}
IMPLEMENTING = set(REDUCTIONS) | {"SET_RESOURCE"}
TERMINAL = {"DIA", "DENSE"}
BRANCHING = {"ROW_DIV", "COL_DIV", "BIN", "DIA_DECOM", "DENSE_DECOM", "HYB_DECOM"}
SORT_FAMILY = {"SORT", "SORT_SUB", "BIN"}
LEVEL_ORDER = {"BMTB": 0, "BMW": 1, "BMT": 2}
RED_ORDER = {"BMT": 0, "BMW": 1, "BMTB": 2, "GMEM": 3}

# name -> ordered list of (key, type, default); type in int|float|ilist|scope
SCHEMA: dict[str, list[tuple[str, str, Any]]] = {
    "ROW_DIV": [("cuts", "ilist", None)],
    "COL_DIV": [("cuts", "ilist", None)],
    "SORT": [],
    "SORT_SUB": [("g", "int", None)],
    "BIN": [("t", "ilist", None)],
    "DIA_DECOM": [("theta", "float", None), ("max", "int", 8)],
    "DENSE_DECOM": [("b", "int", None), ("theta", "float", None)],
    "HYB_DECOM": [("w", "int", None)],   # NEXT-4: the HYB split P:583 names as missing
    "COMPRESS": [],
    "DIA": [],
    "DENSE": [],
    "BMTB_ROW_BLOCK": [("rows", "int", None)],
    "BMTB_NNZ_BLOCK": [("nnz", "int", None)],
    "BMW_ROW_BLOCK": [("rows", "int", None)],
    "BMW_NNZ_BLOCK": [("nnz", "int", None)],
    "BMT_ROW_BLOCK": [("rows", "int", None)],
    "BMT_NNZ_BLOCK": [("nnz", "int", None)],
    "BMT_PAD": [("scope", "scope", "GLOBAL"), ("vec", "int", 0)],
    "SORT_BMTB": [],
    # stages / xcache: shared-memory resource choices of the implementing stage (TMA staging of
    # CSR-stream blocks; x entries staged per CTA); they do not change what y is (R-xcache).
    # stream: the launch stream of the branch's kernel; parts on different streams run
    # concurrently, which changes the writer rule (R-conc, writer_rule in builder_ref)
    "SET_RESOURCE": [("tpb", "int", 256), ("grid", "int", 0), ("stages", "int", 2), ("xcache", "int", 0),
                     ("stream", "int", 0)],
    **{r: [] for r in REDUCTIONS},
}
ALIASES = {"WARP_SEG_RED": "WARP_SEG_ADD_RED", "THREAD_BITMAP_RED": "THREAD_BITMAP_RED_G",
           "SET_RESOURCES": "SET_RESOURCE", "BMTB_ROW_DIV": "BMTB_ROW_BLOCK",
           "THREAD_TOTOAL_RED": "THREAD_TOTAL_RED"}


class GraphParseError(ValueError):
    pass


class GraphIllegal(ValueError):
    def __init__(self, rule: str, node: int, msg: str):
        super().__init__(f"{rule} at node {node}: {msg}")
        self.rule, self.node = rule, node


@dataclasses.dataclass
class Op:
    name: str
    params: dict
    branches: list  # list[list[Op]]


# ------------------------------------------------------------------ parsing
_TOK = re.compile(r"\s*(?:(?P<num>[-+]?(?:\d+\.?\d*|\.\d+)(?:[eE][-+]?\d+)?)|(?P<id>[A-Za-z_][A-Za-z0-9_]*)|(?P<p>[();{}|,=\[\]]))")


def _tokenize(text: str):
    toks, pos = [], 0
    text = text.rstrip()
    while pos < len(text):
        mt = _TOK.match(text, pos)
        if not mt or mt.end() == pos:
            raise GraphParseError(f"bad character at {pos}: {text[pos:pos+10]!r}")
        pos = mt.end()
        if mt.group("num") is not None:
            toks.append(("num", mt.group("num")))
        elif mt.group("id") is not None:
            toks.append(("id", mt.group("id")))
        else:
            toks.append(("p", mt.group("p")))
    toks.append(("eof", ""))
    return toks


def _num(s: str):
    if re.fullmatch(r"[-+]?\d+", s):
        return int(s)
    return float(s)


class _Parser:
    def __init__(self, text):
        self.t = _tokenize(text)
        self.i = 0

    def peek(self):
        return self.t[self.i]

    def take(self, kind=None, val=None):
        tok = self.t[self.i]
        if kind and tok[0] != kind or val is not None and tok[1] != val:
            raise GraphParseError(f"expected {val or kind}, got {tok[1]!r} (token {self.i})")
        self.i += 1
        return tok

    def seq(self):
        ops = [self.op()]
        while self.peek() == ("p", ";"):
            self.take()
            ops.append(self.op())
        return ops

    def value(self):
        tok = self.peek()
        if tok == ("p", "["):
            self.take()
            vals = []
            if self.peek() != ("p", "]"):
                vals.append(_num(self.take("num")[1]))
                while self.peek() == ("p", ","):
                    self.take()
                    vals.append(_num(self.take("num")[1]))
            self.take("p", "]")
            return vals
        if tok[0] == "num":
            return _num(self.take()[1])
        if tok[0] == "id":
            return self.take()[1]
        raise GraphParseError(f"bad value {tok[1]!r}")

    def op(self):
        name = self.take("id")[1]
        name = ALIASES.get(name, name)
        if name not in SCHEMA:
            raise GraphParseError(f"unknown operator {name}")
        schema = SCHEMA[name]
        args_pos, args_kw = [], {}
        if self.peek() == ("p", "("):
            self.take()
            if self.peek() != ("p", ")"):
                while True:
                    if self.peek()[0] == "id" and self.t[self.i + 1] == ("p", "="):
                        key = self.take()[1]
                        self.take()
                        if key in args_kw:
                            raise GraphParseError(f"duplicate key {key}")
                        args_kw[key] = self.value()
                    else:
                        if args_kw:
                            raise GraphParseError("positional after keyword")
                        args_pos.append(self.value())
                    if self.peek() == ("p", ","):
                        self.take()
                        continue
                    break
            self.take("p", ")")
        params = {}
        if len(args_pos) > len(schema):
            raise GraphParseError(f"{name}: too many arguments")
        for (key, _, _), v in zip(schema, args_pos):
            params[key] = v
        for key, v in args_kw.items():
            if key not in {k for k, _, _ in schema}:
                raise GraphParseError(f"{name}: unknown parameter {key}")
            if key in params:
                raise GraphParseError(f"{name}: {key} given twice")
            params[key] = v
        for key, typ, default in schema:
            if key not in params:
                if default is None:
                    raise GraphParseError(f"{name}: missing parameter {key}")
                params[key] = default
            params[key] = _coerce(name, key, typ, params[key])
        branches = []
        if self.peek() == ("p", "{"):
            self.take()
            branches.append(self.seq())
            while self.peek() == ("p", "|"):
                self.take()
                branches.append(self.seq())
            self.take("p", "}")
        return Op(name, params, branches)


def _coerce(name, key, typ, v):
    if typ == "int":
        if isinstance(v, float) and v.is_integer():
            v = int(v)
        if not isinstance(v, int):
            raise GraphParseError(f"{name}.{key}: integer expected")
        return v
    if typ == "float":
        if isinstance(v, (int, float)) and not isinstance(v, bool):
            return float(v)
        raise GraphParseError(f"{name}.{key}: number expected")
    if typ == "ilist":
        if not isinstance(v, list):
            v = [v] if isinstance(v, int) else v
        if not isinstance(v, list) or not all(isinstance(a, int) or (isinstance(a, float) and a.is_integer()) for a in v):
            raise GraphParseError(f"{name}.{key}: integer list expected")
        return [int(a) for a in v]
    if typ == "scope":
        if v not in ("GLOBAL", "BMTB", "BMW"):
            raise GraphParseError(f"{name}.{key}: GLOBAL|BMTB|BMW expected")
        return v
    raise AssertionError(typ)


def n_branches(op: Op) -> int:
    if op.name in ("ROW_DIV", "COL_DIV"):
        return len(op.params["cuts"]) + 1
    if op.name == "BIN":
        return len(op.params["t"]) + 1
    if op.name in ("DIA_DECOM", "DENSE_DECOM", "HYB_DECOM"):
        return 2
    return 0


def parse(text: str) -> list:
    """Parse + expand replicated branches; raise GraphParseError or GraphIllegal."""
    p = _Parser(text)
    g = p.seq()
    p.take("eof")
    _expand(g)
    validate(g)
    return g


def _expand(seq):
    for op in seq:
        for b in op.branches:
            _expand(b)
        if op.name in ("ROW_DIV", "COL_DIV", "BIN", "HYB_DECOM") and len(op.branches) == 1:
            k = n_branches(op)
            op.branches = [_clone(op.branches[0]) for _ in range(k)]


def _clone(seq):
    return [Op(o.name, dict((k, list(v) if isinstance(v, list) else v) for k, v in o.params.items()),
               [_clone(b) for b in o.branches]) for o in seq]


# ------------------------------------------------------------------ printing
def _fmt(v):
    if isinstance(v, list):
        return "[" + ",".join(str(a) for a in v) + "]"
    if isinstance(v, float):
        return repr(v)
    return str(v)


def to_string(seq) -> str:
    out = []
    for op in seq:
        s = op.name
        if SCHEMA[op.name]:
            # SET_RESOURCE stream (R-conc) is printed only when non-zero
            s += "(" + ",".join(f"{k}={_fmt(op.params[k])}" for k, _, _ in SCHEMA[op.name]
                                if not (k == "stream" and op.params[k] == 0)) + ")"
        if op.branches:
            s += " { " + " | ".join(to_string(b) for b in op.branches) + " }"
        out.append(s)
    return "; ".join(out)


# ------------------------------------------------------------------ validation (A16)
def _check_params(op: Op, nid: int):
    p = op.params

    def bad(msg):
        raise GraphIllegal("PARAM", nid, f"{op.name}: {msg}")
    if op.name in ("ROW_DIV", "COL_DIV"):
        c = p["cuts"]
        if not c or c[0] <= 0 or any(b <= a for a, b in zip(c, c[1:])):
            bad("cuts must be non-empty, positive, strictly increasing")
    elif op.name == "BIN":
        t = p["t"]
        if not t or t[0] < 1 or any(b <= a for a, b in zip(t, t[1:])):
            bad("thresholds must be non-empty, >= 1, strictly ascending")
    elif op.name == "SORT_SUB":
        if p["g"] < 2:
            bad("g >= 2")
    elif op.name == "DIA_DECOM":
        if not (0.0 < p["theta"] <= 1.0) or p["max"] < 1:
            bad("0 < theta <= 1, max >= 1")
    elif op.name == "DENSE_DECOM":
        if not (0.0 < p["theta"] <= 1.0) or p["b"] < 1:
            bad("0 < theta <= 1, b >= 1")
    elif op.name == "HYB_DECOM":
        if p["w"] < 1:
            bad("w >= 1")
    elif op.name.endswith("_BLOCK"):
        v = p.get("rows", p.get("nnz"))
        if v < 1:
            bad("block size >= 1")
    elif op.name == "BMT_PAD":
        if p["vec"] not in (0, 1, 2, 4):
            bad("vec in {0,1,2,4}")
    elif op.name == "SET_RESOURCE":
        if (p["tpb"] < 32 or p["tpb"] > 1024 or p["tpb"] % 32 or p["grid"] < 0 or p["stages"] not in (0, 2)
                or not 0 <= p["xcache"] <= 65536 or not 0 <= p["stream"] <= 3):
            bad("tpb multiple of 32 in [32,1024], grid >= 0, stages in {0,2}, xcache in [0,65536], stream in [0,3]")


def validate(seq):
    """Raise GraphIllegal for the first violated rule (pre-order node ids)."""
    counter = [0]
    ids = {}

    def number(s):
        for op in s:
            ids[id(op)] = counter[0]
            counter[0] += 1
            for b in op.branches:
                number(b)
    number(seq)
    _walk(seq, [], ids)


def _walk(seq, prefix, ids):
    for k, op in enumerate(seq):
        nid = ids[id(op)]
        _check_params(op, nid)
        if op.name in BRANCHING:
            if k != len(seq) - 1:
                raise GraphIllegal("R8", nid, "a branching operator must end its sequence")
            nb = n_branches(op)
            if op.name in ("DIA_DECOM", "DENSE_DECOM"):
                if len(op.branches) not in (1, 2):
                    raise GraphIllegal("R8", nid, "DIA/DENSE_DECOM take 1 or 2 branches")
            elif len(op.branches) != nb:
                raise GraphIllegal("R8", nid, f"expected {nb} branches, got {len(op.branches)}")
            path = prefix + list(seq[:k + 1])
            _check_path(path, ids, partial=True)
            for bi, b in enumerate(op.branches):
                if op.name in ("DIA_DECOM", "DENSE_DECOM") and bi == 0:
                    _check_terminal(op, b, ids)
                else:
                    if b and b[0].name in TERMINAL:
                        raise GraphIllegal("R8", ids[id(b[0])], "DIA/DENSE only open the first decomposition branch")
                    _walk(b, path, ids)
            return
        if op.branches:
            raise GraphIllegal("R8", nid, f"{op.name} does not branch")
        if op.name in TERMINAL:
            raise GraphIllegal("R8", nid, "DIA/DENSE only open the first decomposition branch")
    _check_path(prefix + list(seq), ids, partial=False)


def _check_terminal(dec: Op, b, ids):
    want = "DIA" if dec.name == "DIA_DECOM" else "DENSE"
    if not b or b[0].name != want:
        raise GraphIllegal("R8", ids[id(dec)], f"first branch must start with {want}")
    for op in b[1:]:
        if op.name != "SET_RESOURCE" or op.branches:
            raise GraphIllegal("R8", ids[id(op)], f"{want} branch admits only SET_RESOURCE")
        _check_params(op, ids[id(op)])
    if len(b) > 2:
        raise GraphIllegal("R9", ids[id(b[2])], "at most one SET_RESOURCE")


def _stage(name):
    if name in CONVERTING:
        return 0
    if name == "COMPRESS":
        return 1
    if name in MAPPING:
        return 2
    return 3


def _check_path(path, ids, partial):
    stage = 0
    n_compress = 0
    seen_conv = set()
    levels = []          # blocking levels in order
    level_kind = {}
    reds = []
    n_set = 0
    pad = sort_bmtb = False
    sorted_ = False
    for op in path:
        nid = ids[id(op)]
        st = _stage(op.name)
        if st >= 2 and n_compress == 0:
            raise GraphIllegal("R1", nid, f"{op.name} before COMPRESS")
        if st < stage or (st == 1 and stage >= 1):
            raise GraphIllegal("R1", nid, f"{op.name} out of stage order")
        stage = st
        if st == 0:
            if op.name in seen_conv:
                raise GraphIllegal("R11", nid, f"{op.name} twice on a path")
            if op.name in SORT_FAMILY and seen_conv & SORT_FAMILY:
                raise GraphIllegal("R11", nid, "SORT/SORT_SUB/BIN are mutually exclusive")
            if op.name in ("DIA_DECOM", "DENSE_DECOM") and sorted_:
                raise GraphIllegal("R10", nid, f"{op.name} after a row permutation")
            if op.name in SORT_FAMILY:
                sorted_ = True
            seen_conv.add(op.name)
        elif st == 1:
            n_compress += 1
        elif st == 2:
            if op.name.endswith("_BLOCK"):
                lvl = op.name.split("_")[0]
                if lvl in level_kind:
                    raise GraphIllegal("R4", nid, f"second {lvl} blocking")
                if levels and LEVEL_ORDER[levels[-1]] > LEVEL_ORDER[lvl]:
                    raise GraphIllegal("R3", nid, f"{lvl} after {levels[-1]}")
                if pad:
                    raise GraphIllegal("R5", nid, "blocking after BMT_PAD")
                levels.append(lvl)
                level_kind[lvl] = op.name.split("_")[1]
            elif op.name == "BMT_PAD":
                if pad:
                    raise GraphIllegal("R5", nid, "BMT_PAD twice")
                if "BMT" not in level_kind:
                    raise GraphIllegal("R5", nid, "BMT_PAD needs BMT blocking")
                sc = op.params["scope"]
                if sc != "GLOBAL" and sc not in level_kind:
                    raise GraphIllegal("R5", nid, f"BMT_PAD scope {sc} needs {sc} blocking")
                pad = True
            elif op.name == "SORT_BMTB":
                if sort_bmtb:
                    raise GraphIllegal("R5", nid, "SORT_BMTB twice")
                if level_kind.get("BMTB") != "ROW" or "BMW" in level_kind or "BMT" in level_kind:
                    raise GraphIllegal("R5", nid, "SORT_BMTB needs BMTB_ROW_BLOCK and precedes BMW/BMT")
                sort_bmtb = True
        else:
            if op.name == "SET_RESOURCE":
                n_set += 1
                if n_set > 1:
                    raise GraphIllegal("R9", nid, "SET_RESOURCE twice")
                continue
            lvl = REDUCTIONS[op.name]
            if lvl != "GMEM" and lvl not in level_kind:
                raise GraphIllegal("R6", nid, f"{op.name} needs {lvl} blocking")
            if reds and RED_ORDER[reds[-1]] >= RED_ORDER[lvl]:
                raise GraphIllegal("R6", nid, f"{op.name} out of reduction order")
            reds.append(lvl)
    if partial:
        if n_compress:
            raise GraphIllegal("R1", ids[id(path[-1])], "branching after COMPRESS")
        return
    last = path[-1] if path else None
    nid = ids[id(last)] if last is not None else 0
    if n_compress != 1:
        raise GraphIllegal("R2", nid, "path needs exactly one COMPRESS")
    if not reds or reds[-1] != "GMEM":
        raise GraphIllegal("R7", nid, "path must end with GMEM_ATOM_RED")
    if last.name != "GMEM_ATOM_RED":
        # SET_RESOURCE may not follow GMEM (GMEM is the terminal token, R7)
        raise GraphIllegal("R7", nid, "GMEM_ATOM_RED must be the last operator")


def is_legal(text: str) -> bool:
    try:
        parse(text)
        return True
    except (GraphParseError, GraphIllegal):
        return False
