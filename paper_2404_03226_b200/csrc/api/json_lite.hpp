// json_lite.hpp -- minimal JSON reader/writer for the two host file formats
// of the API (NDJSON DAG records, platform JSON).  Objects keep insertion
// order so records serialize byte-stably ("kind" first).
#pragma once

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace tbsim_json {

struct ParseError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct Value {
    enum Type { Null, Bool, Int, Double, String, Array, Object } type = Null;
    bool b = false;
    std::int64_t i = 0;
    double d = 0.0;
    std::string s;
    std::vector<Value> arr;
    std::vector<std::pair<std::string, Value>> obj;

    bool is_number() const { return type == Int || type == Double; }
    bool is_integer() const { return type == Int; }
    double number() const { return type == Int ? static_cast<double>(i) : d; }
    const Value* find(const std::string& key) const {
        for (const auto& kv : obj)
            if (kv.first == key) return &kv.second;
        return nullptr;
    }
};

class Parser {
public:
    explicit Parser(const std::string& text) : t_(text) {}
    Value parse_document() {
        ws();
        Value v = value();
        ws();
        if (p_ != t_.size()) err("unexpected trailing characters");
        return v;
    }

private:
    [[noreturn]] void err(const std::string& what) const {
        throw ParseError("syntax error at byte " + std::to_string(p_ + 1) + ": " + what);
    }
    void ws() {
        while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\t' || t_[p_] == '\n' || t_[p_] == '\r')) ++p_;
    }
    char peek() const { return p_ < t_.size() ? t_[p_] : '\0'; }
    void expect(char c) {
        if (peek() != c) err(std::string("expected '") + c + "'");
        ++p_;
    }
    Value value() {
        ws();
        const char c = peek();
        if (c == '{') return object();
        if (c == '[') return array();
        if (c == '"') {
            Value v;
            v.type = Value::String;
            v.s = string();
            return v;
        }
        if (c == '-' || (c >= '0' && c <= '9')) return number();
        if (t_.compare(p_, 4, "true") == 0) { p_ += 4; Value v; v.type = Value::Bool; v.b = true; return v; }
        if (t_.compare(p_, 5, "false") == 0) { p_ += 5; Value v; v.type = Value::Bool; return v; }
        if (t_.compare(p_, 4, "null") == 0) { p_ += 4; return Value{}; }
        err("invalid literal");
    }
    Value object() {
        Value v;
        v.type = Value::Object;
        expect('{');
        ws();
        if (peek() == '}') { ++p_; return v; }
        for (;;) {
            ws();
            if (peek() != '"') err("expected object key");
            std::string k = string();
            ws();
            expect(':');
            Value x = value();
            v.obj.emplace_back(std::move(k), std::move(x));
            ws();
            if (peek() == ',') { ++p_; continue; }
            expect('}');
            return v;
        }
    }
    Value array() {
        Value v;
        v.type = Value::Array;
        expect('[');
        ws();
        if (peek() == ']') { ++p_; return v; }
        for (;;) {
            v.arr.push_back(value());
            ws();
            if (peek() == ',') { ++p_; continue; }
            expect(']');
            return v;
        }
    }
    std::string string() {
        expect('"');
        std::string out;
        while (p_ < t_.size() && t_[p_] != '"') {
            char c = t_[p_++];
            if (c == '\\') {
                if (p_ >= t_.size()) err("bad escape");
                const char e = t_[p_++];
                switch (e) {
                    case '"': out += '"'; break;
                    case '\\': out += '\\'; break;
                    case '/': out += '/'; break;
                    case 'b': out += '\b'; break;
                    case 'f': out += '\f'; break;
                    case 'n': out += '\n'; break;
                    case 'r': out += '\r'; break;
                    case 't': out += '\t'; break;
                    case 'u': {
                        if (p_ + 4 > t_.size()) err("bad unicode escape");
                        const unsigned cp = static_cast<unsigned>(std::stoul(t_.substr(p_, 4), nullptr, 16));
                        p_ += 4;
                        if (cp < 0x80) out += static_cast<char>(cp);
                        else if (cp < 0x800) { out += static_cast<char>(0xC0 | (cp >> 6)); out += static_cast<char>(0x80 | (cp & 0x3F)); }
                        else { out += static_cast<char>(0xE0 | (cp >> 12)); out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F)); out += static_cast<char>(0x80 | (cp & 0x3F)); }
                        break;
                    }
                    default: err("bad escape");
                }
            } else if (static_cast<unsigned char>(c) < 0x20) {
                err("control character in string");
            } else {
                out += c;
            }
        }
        expect('"');
        return out;
    }
    Value number() {
        const size_t start = p_;
        if (peek() == '-') ++p_;
        if (!(peek() >= '0' && peek() <= '9')) err("bad number");
        while (peek() >= '0' && peek() <= '9') ++p_;
        bool real = false;
        if (peek() == '.') {
            real = true;
            ++p_;
            if (!(peek() >= '0' && peek() <= '9')) err("bad number");
            while (peek() >= '0' && peek() <= '9') ++p_;
        }
        if (peek() == 'e' || peek() == 'E') {
            real = true;
            ++p_;
            if (peek() == '+' || peek() == '-') ++p_;
            if (!(peek() >= '0' && peek() <= '9')) err("bad number");
            while (peek() >= '0' && peek() <= '9') ++p_;
        }
        Value v;
        const std::string tok = t_.substr(start, p_ - start);
        if (!real) {
            try {
                v.type = Value::Int;
                v.i = std::stoll(tok);
                return v;
            } catch (const std::out_of_range&) {
                real = true;
            }
        }
        v.type = Value::Double;
        v.d = std::stod(tok);
        return v;
    }
    const std::string& t_;
    size_t p_ = 0;
};

inline Value parse(const std::string& text) { return Parser(text).parse_document(); }

inline void dump_string(std::string& out, const std::string& s) {
    out += '"';
    for (const char c : s) {
        switch (c) {
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            case '\b': out += "\\b"; break;
            case '\f': out += "\\f"; break;
            case '\n': out += "\\n"; break;
            case '\r': out += "\\r"; break;
            case '\t': out += "\\t"; break;
            default:
                if (static_cast<unsigned char>(c) < 0x20) {
                    char buf[8];
                    std::snprintf(buf, sizeof buf, "\\u%04x", static_cast<unsigned char>(c));
                    out += buf;
                } else {
                    out += c;
                }
        }
    }
    out += '"';
}

}  // namespace tbsim_json
