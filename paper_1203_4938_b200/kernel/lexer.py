"""Tokenizer (SPEC kernel-lang: tokenize), total ``scan`` + strict ``tokenize``."""

from __future__ import annotations

from dataclasses import dataclass

from ..errors import KernelError

__all__ = ["Token", "scan", "tokenize", "KernelLexError"]


class KernelLexError(KernelError):
    """Illegal character (with position)."""


KEYWORDS = frozenset({"if", "else", "for"})
# two-character operators are tried before their one-character prefixes
_OPS2 = ("<<", ">>", "<=", ">=", "==", "!=", "&&", "||")
_OPS1 = frozenset("+-*/%<>=!~&|^?:;,.()[]{}")


@dataclass(frozen=True)
class Token:
    kind: str  # identifier | int | float | punct | keyword | error
    lexeme: str
    line: int
    col: int
    value: object = None


def _number(src: str, i: int) -> tuple[str, str, object]:
    """(kind, lexeme, value) of the numeric literal starting at i."""
    n = len(src)
    if src[i] == "0" and i + 1 < n and src[i + 1] in "xX":
        j = i + 2
        while j < n and src[j] in "0123456789abcdefABCDEF":
            j += 1
        text = src[i:j]
        return ("int", text, int(text, 16)) if j > i + 2 else ("error", text, None)
    j = i
    while j < n and src[j].isdigit():
        j += 1
    is_float = False
    if j < n and src[j] == ".":
        is_float = True
        j += 1
        while j < n and src[j].isdigit():
            j += 1
    if j < n and src[j] in "eE":
        k = j + 1
        if k < n and src[k] in "+-":
            k += 1
        if k < n and src[k].isdigit():
            is_float = True
            j = k
            while j < n and src[j].isdigit():
                j += 1
    if j < n and src[j] in "fF":
        is_float = True
        text = src[i:j + 1]
        return "float", text, float(src[i:j])
    text = src[i:j]
    return ("float", text, float(text)) if is_float else ("int", text, int(text))


def scan(source: str) -> list[Token]:
    out: list[Token] = []
    i, line, col, n = 0, 1, 1, len(source)

    def move(text: str) -> None:
        nonlocal line, col
        nl = text.count("\n")
        if nl:
            line += nl
            col = len(text) - text.rfind("\n")
        else:
            col += len(text)

    while i < n:
        c = source[i]
        if c in " \t\r\n":
            move(c)
            i += 1
        elif source.startswith("//", i):
            j = source.find("\n", i)
            j = n if j < 0 else j
            move(source[i:j])
            i = j
        elif source.startswith("/*", i):
            j = source.find("*/", i + 2)
            if j < 0:
                out.append(Token("error", source[i:], line, col))
                move(source[i:])
                i = n
            else:
                move(source[i:j + 2])
                i = j + 2
        elif c.isalpha() or c == "_":
            j = i + 1
            while j < n and (source[j].isalnum() or source[j] == "_"):
                j += 1
            text = source[i:j]
            out.append(Token("keyword" if text in KEYWORDS else "identifier", text, line, col))
            move(text)
            i = j
        elif c.isdigit() or (c == "." and i + 1 < n and source[i + 1].isdigit()):
            kind, text, value = _number(source, i)
            out.append(Token(kind, text, line, col, value))
            move(text)
            i += len(text)
        elif source[i:i + 2] in _OPS2:
            out.append(Token("punct", source[i:i + 2], line, col))
            move(source[i:i + 2])
            i += 2
        elif c in _OPS1:
            out.append(Token("punct", c, line, col))
            move(c)
            i += 1
        else:
            out.append(Token("error", c, line, col))
            move(c)
            i += 1
    return out


def tokenize(source: str) -> list[Token]:
    toks = scan(source)
    for t in toks:
        if t.kind == "error":
            raise KernelLexError(f"illegal character {t.lexeme[:1]!r}", t.line, t.col)
    return toks
