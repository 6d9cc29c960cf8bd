#pragma once
// Minimal CSV helpers shared by the catalog and trace readers. Field rules of
// the reference readers (proj/src/catalog.cpp:28-41): split on ',', drop '\r',
// no quoting.
#include <cstdint>
#include <istream>
#include <stdexcept>
#include <string>
#include <vector>

namespace gpufaas::csv {

inline std::vector<std::string> split(const std::string& line) {
    std::vector<std::string> out(1);
    for (char c : line) {
        if (c == ',') out.emplace_back();
        else if (c != '\r') out.back().push_back(c);
    }
    return out;
}

inline bool blank(const std::string& line) { return line.empty() || line == "\r"; }

class LineReader {
public:
    LineReader(std::istream& in, std::string origin) : in_(in), origin_(std::move(origin)) {}
    bool next(std::string& line) {
        if (!std::getline(in_, line)) return false;
        ++lineno_;
        return true;
    }
    std::runtime_error error(const std::string& what) const {
        return std::runtime_error(origin_ + ":" + std::to_string(lineno_) + ": " + what);
    }
    double number(const std::string& field, const std::string& name) const {
        std::size_t used = 0;
        double v = 0;
        bool ok = true;
        try {
            v = std::stod(field, &used);
        } catch (const std::exception&) {
            ok = false;
        }
        if (!ok || used != field.size()) throw error("bad " + name + " value '" + field + "'");
        return v;
    }
    std::int64_t count(const std::string& field) const {
        std::size_t used = 0;
        long long v = -1;
        bool ok = true;
        try {
            v = std::stoll(field, &used);
        } catch (const std::exception&) {
            ok = false;
        }
        if (!ok || used != field.size() || v < 0) throw error("bad count '" + field + "'");
        return v;
    }

private:
    std::istream& in_;
    std::string origin_;
    std::size_t lineno_ = 0;
};

}  // namespace gpufaas::csv
