"""Oracle-side parser for the protobuf-text scene format (TEST INFRASTRUCTURE).

Independent of the library's C++ parser (paper_2106_13281_b200/csrc/config.cpp):
the two share no code, and tests compare their integer tables bit for bit.

The grammar is the ProtoBuf text subset the paper exhibits in App. A
("substeps: 1 / dt: .01 / gravity { z: -9.8 } / bodies { ... }"):

    file   := field*
    field  := NAME ':' scalar  |  NAME ':'? '{' field* '}'
    scalar := NUMBER | "STRING" | NAME            (NAME covers true/false)

'#' starts a comment to end of line; ',' and ';' between fields are ignored
(as in protobuf text format).  Numbers follow protobuf text: ".01", "-9.8",
"1e4" are valid.

Result: a list of (name, value, line, col) where value is a float, a str,
a bool, or a nested list of the same shape.
"""
from __future__ import annotations

import re

__all__ = ["ParseError", "parse_text"]


class ParseError(ValueError):
    def __init__(self, line: int, col: int, msg: str):
        super().__init__(f"{line}:{col}: {msg}")
        self.line, self.col, self.msg = line, col, msg


_TOKEN = re.compile(
    r"""
    (?P<ws>[ \t\r\n]+|\#[^\n]*|[,;])
  | (?P<str>"(?:[^"\\\n]|\\.)*")
  | (?P<num>[-+]?(?:\d+\.?\d*|\.\d+)(?:[eE][-+]?\d+)?)
  | (?P<name>[A-Za-z_][A-Za-z0-9_]*)
  | (?P<punct>[:{}])
    """,
    re.VERBOSE,
)


def _tokens(text: str):
    pos, line, line_start = 0, 1, 0
    while pos < len(text):
        m = _TOKEN.match(text, pos)
        col = pos - line_start + 1
        if m is None:
            raise ParseError(line, col, f"unexpected character {text[pos]!r}")
        kind = m.lastgroup
        tok = m.group(kind)
        if kind != "ws":
            yield kind, tok, line, col
        nl = tok.count("\n")
        if nl:
            line += nl
            line_start = m.start() + tok.rfind("\n") + 1
        pos = m.end()
    yield "eof", "", line, pos - line_start + 1


def parse_text(text: str):
    toks = list(_tokens(text))
    i = 0

    def block(top: bool):
        nonlocal i
        out = []
        while True:
            kind, tok, line, col = toks[i]
            if kind == "eof":
                if not top:
                    raise ParseError(line, col, "unexpected end of input: missing '}'")
                return out
            if kind == "punct" and tok == "}":
                if top:
                    raise ParseError(line, col, "unbalanced '}'")
                i += 1
                return out
            if kind != "name":
                raise ParseError(line, col, f"expected field name, got {tok!r}")
            name = tok
            i += 1
            kind, tok, l2, c2 = toks[i]
            if kind == "punct" and tok == ":":
                i += 1
                kind, tok, l2, c2 = toks[i]
                if kind == "punct" and tok == "{":
                    i += 1
                    out.append((name, block(False), line, col))
                    continue
                if kind == "num":
                    val = float(tok)
                elif kind == "str":
                    val = bytes(tok[1:-1], "utf-8").decode("unicode_escape")
                elif kind == "name" and tok in ("true", "false"):
                    val = tok == "true"
                elif kind == "name":
                    val = tok  # enum-like bare identifier
                else:
                    raise ParseError(l2, c2, f"expected value after ':', got {tok!r}")
                i += 1
                out.append((name, val, line, col))
            elif kind == "punct" and tok == "{":
                i += 1
                out.append((name, block(False), line, col))
            else:
                raise ParseError(l2, c2, f"expected ':' or '{{' after {name!r}")

    return block(True)
