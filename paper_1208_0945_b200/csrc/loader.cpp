// loader.cpp -- the era-level long format straight into a device-resident
// dataset: read_long_format (io.hpp:88-174) followed by build_dataset
// (dataset.hpp:74-152), SURVEY §8(f) #3.
//
// The reference reads line by line into a vector<SubjectRecord> and then
// lays out the CSC on the host (minutes and tens of GB at 150M eras, SURVEY
// §8(f)).  Here the file is read once, parsed in parallel chunks split at
// line boundaries, the drug labels are numbered in first-appearance order
// by a merge over the chunks' local label lists, and the pairs (drug, row,
// subject) are emitted in row order and turned into CSC columns on the
// device by a stable sort on the drug (dataset_from_row_pairs).  Every
// error the reference raises is raised here with the same message, and when
// a file holds several errors the one on the earliest line wins, as it does
// for the reference's sequential reader.
#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "engine.h"

namespace bsccs_b200 {

namespace {

struct LineRec {
    std::string_view subject;
    int32_t length, events;
    uint32_t first_label, nlabels; // into the chunk's label-occurrence list
    long line;                     // 1-based line number within the chunk
};

struct Chunk {
    const char* begin = nullptr;
    const char* end = nullptr;
    long lines = 0; // physical lines in the chunk
    std::vector<LineRec> recs;
    std::vector<int32_t> occ;                 // label occurrences (local label ids), per line
    std::vector<std::string_view> labels;     // local labels in first-appearance order
    long err_line = -1;                       // first error within the chunk (local line number)
    std::string err_msg;                      // message without the "path:line: " prefix
    // subject of the failing line when its error comes after the reference's
    // contiguity check (io.hpp:123-132 runs before parse_day and the labels):
    // that check still has precedence on the same line
    std::string_view err_subject;
};

bool parse_int(std::string_view f, int32_t& v) {
    const auto r = std::from_chars(f.data(), f.data() + f.size(), v);
    return r.ec == std::errc() && r.ptr == f.data() + f.size();
}

// Parses one chunk's lines (detail::split_tabs / parse_day / next_line, io.hpp:25-78).
void parse_chunk(Chunk& ch, const std::unordered_map<std::string_view, int32_t>* dict) {
    std::unordered_map<std::string_view, int32_t> local;
    std::vector<std::string_view> fields;
    std::vector<int32_t> era;
    const char* p = ch.begin;
    long line_no = 0;
    auto fail_at = [&](long ln, std::string msg, std::string_view subject = {}) {
        ch.err_line = ln;
        ch.err_msg = std::move(msg);
        ch.err_subject = subject;
        // count the remaining lines: later chunks number theirs after these
        long n = ln;
        const char* q = p;
        while (q < ch.end) {
            const char* nl = static_cast<const char*>(std::memchr(q, '\n', static_cast<size_t>(ch.end - q)));
            ++n;
            q = nl ? nl + 1 : ch.end;
        }
        ch.lines = n;
    };
    while (p < ch.end) {
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(ch.end - p)));
        const char* le = nl ? nl : ch.end;
        ++line_no;
        std::string_view line(p, static_cast<size_t>(le - p));
        p = nl ? nl + 1 : ch.end;
        if (!line.empty() && line.back() == '\r') line.remove_suffix(1);
        if (line.empty()) continue;
        fields.clear();
        size_t start = 0;
        for (size_t q = 0; q <= line.size(); ++q) {
            if (q == line.size() || line[q] == '\t') {
                fields.push_back(line.substr(start, q - start));
                start = q + 1;
            }
        }
        if (fields.size() != 3 && fields.size() != 4) return fail_at(line_no, "expected 3 or 4 tab-separated fields");
        if (fields[0].empty()) return fail_at(line_no, "empty subject id");
        LineRec r;
        r.subject = fields[0];
        r.line = line_no;
        if (!parse_int(fields[1], r.length))
            return fail_at(line_no, "expected an integer, got '" + std::string(fields[1]) + "'", r.subject);
        if (!parse_int(fields[2], r.events))
            return fail_at(line_no, "expected an integer, got '" + std::string(fields[2]) + "'", r.subject);
        r.first_label = static_cast<uint32_t>(ch.occ.size());
        era.clear();
        if (fields.size() == 4 && !fields[3].empty()) {
            std::string_view rest = fields[3];
            while (!rest.empty()) {
                const size_t sp = rest.find(' ');
                const std::string_view label = rest.substr(0, sp);
                rest = sp == std::string_view::npos ? std::string_view{} : rest.substr(sp + 1);
                if (label.empty()) continue; // tolerate doubled separators
                if (dict) {
                    const auto f = dict->find(label);
                    if (f == dict->end())
                        return fail_at(line_no, "drug '" + std::string(label) + "' is not in the dictionary",
                                       r.subject);
                    era.push_back(f->second);
                } else {
                    auto f = local.find(label);
                    if (f == local.end()) {
                        f = local.emplace(label, static_cast<int32_t>(ch.labels.size())).first;
                        ch.labels.push_back(label);
                    }
                    era.push_back(f->second);
                }
            }
            // duplicates: the same label twice (equal ids <=> equal labels)
            std::vector<int32_t> sorted(era);
            std::sort(sorted.begin(), sorted.end());
            for (size_t k = 1; k < sorted.size(); ++k)
                if (sorted[k] == sorted[k - 1]) return fail_at(line_no, "drug listed twice in one era", r.subject);
        }
        ch.occ.insert(ch.occ.end(), era.begin(), era.end());
        r.nlabels = static_cast<uint32_t>(era.size());
        ch.recs.push_back(r);
    }
    ch.lines = line_no;
}

} // namespace

bsccs_dataset* load_long_format(const char* path, const char* const* dictionary, int32_t dict_size, int device,
                                int ctas_override, int threads) {
    NvtxRange nvtx_("read_long_format");
    if (!path) input_error("read_long_format: null path");
    const std::string spath(path);
    // ---- the file -------------------------------------------------------
    std::FILE* f = std::fopen(path, "rb");
    if (!f) input_error("cannot open '" + spath + "' for reading");
    std::vector<char> buf;
    {
        std::fseek(f, 0, SEEK_END);
        const long n = std::ftell(f);
        std::fseek(f, 0, SEEK_SET);
        buf.resize(static_cast<size_t>(std::max(n, 0L)));
        const size_t got = n > 0 ? std::fread(buf.data(), 1, buf.size(), f) : 0;
        std::fclose(f);
        if (got != buf.size()) input_error("cannot open '" + spath + "' for reading");
    }
    // ---- dictionary -------------------------------------------------------
    std::vector<std::string> drug_ids;
    std::unordered_map<std::string_view, int32_t> dict;
    const bool fixed = dictionary && dict_size > 0;
    if (fixed) {
        drug_ids.reserve(static_cast<size_t>(dict_size));
        for (int32_t j = 0; j < dict_size; ++j) drug_ids.emplace_back(dictionary[j] ? dictionary[j] : "");
        for (int32_t j = 0; j < dict_size; ++j)
            if (!dict.emplace(drug_ids[static_cast<size_t>(j)], j).second)
                input_error("duplicate drug label '" + drug_ids[static_cast<size_t>(j)] + "' in dictionary");
    }
    // ---- parallel parse over line-aligned chunks ---------------------------
    unsigned T = threads > 0 ? static_cast<unsigned>(threads) : std::max(1u, std::thread::hardware_concurrency());
    T = static_cast<unsigned>(std::min<size_t>(T, std::max<size_t>(1, buf.size() >> 20)));
    std::vector<Chunk> chunks(T);
    {
        const char* b = buf.data();
        const char* e = b + buf.size();
        const char* cur = b;
        for (unsigned t = 0; t < T; ++t) {
            chunks[t].begin = cur;
            const char* target = t + 1 == T ? e : b + buf.size() * (t + 1) / T;
            if (target < cur) target = cur;
            if (t + 1 < T && target < e) {
                const char* nl = static_cast<const char*>(std::memchr(target, '\n', static_cast<size_t>(e - target)));
                target = nl ? nl + 1 : e;
            }
            chunks[t].end = target;
            cur = target;
        }
    }
    {
        std::vector<std::thread> th;
        for (unsigned t = 0; t < T; ++t) th.emplace_back(parse_chunk, std::ref(chunks[t]), fixed ? &dict : nullptr);
        for (auto& x : th) x.join();
    }
    // global line numbers (every chunk counted all of its lines)
    std::vector<long> line_base(T, 0);
    for (unsigned t = 1; t < T; ++t) line_base[t] = line_base[t - 1] + chunks[t - 1].lines;
    // the earliest line-local error (parse, field count, dictionary, duplicate)
    long first_err = -1;
    std::string first_msg;
    std::string_view first_subject;
    for (unsigned t = 0; t < T && first_err < 0; ++t)
        if (chunks[t].err_line >= 0) {
            first_err = line_base[t] + chunks[t].err_line;
            first_msg = chunks[t].err_msg;
            first_subject = chunks[t].err_subject;
        }
    // labels numbered in first-appearance order (chunk order = file order)
    std::vector<std::vector<int32_t>> remap(T);
    if (!fixed) {
        std::unordered_map<std::string_view, int32_t> global;
        for (unsigned t = 0; t < T; ++t) {
            remap[t].resize(chunks[t].labels.size());
            for (size_t k = 0; k < chunks[t].labels.size(); ++k) {
                auto it = global.find(chunks[t].labels[k]);
                if (it == global.end()) {
                    it = global.emplace(chunks[t].labels[k], static_cast<int32_t>(drug_ids.size())).first;
                    drug_ids.emplace_back(chunks[t].labels[k]);
                }
                remap[t][k] = it->second;
            }
        }
    }
    // records: runs of consecutive lines of one subject; a subject seen again
    // later is an error (its rows must be contiguous) -- scanned in file order
    // up to the earliest line-local error
    std::vector<std::pair<unsigned, uint32_t>> line_order; // (chunk, line record) in file order
    std::vector<int64_t> rec_start;                          // into line_order
    {
        std::unordered_set<std::string_view> seen;
        std::string_view last;
        bool have = false, stop = false;
        for (unsigned t = 0; t < T && !stop; ++t) {
            for (uint32_t i = 0; i < chunks[t].recs.size(); ++i) {
                const LineRec& r = chunks[t].recs[i];
                const long gline = line_base[t] + r.line;
                if (first_err >= 0 && gline >= first_err) {
                    stop = true;
                    break;
                }
                if (!have || r.subject != last) {
                    if (!seen.insert(r.subject).second) {
                        first_err = gline;
                        first_msg = "rows of subject '" + std::string(r.subject) + "' are not contiguous";
                        stop = true;
                        break;
                    }
                    rec_start.push_back(static_cast<int64_t>(line_order.size()));
                    last = r.subject;
                    have = true;
                }
                line_order.emplace_back(t, i);
            }
        }
        // the failing line itself: the contiguity check precedes its error
        if (!stop && first_err >= 0 && !first_subject.empty() && (!have || first_subject != last) &&
            seen.count(first_subject))
            first_msg = "rows of subject '" + std::string(first_subject) + "' are not contiguous";
    }
    if (first_err >= 0) input_error(spath + ":" + std::to_string(first_err) + ": " + first_msg);
    rec_start.push_back(static_cast<int64_t>(line_order.size()));

    // ---- build_dataset (dataset.hpp:74-152) ----------------------------------
    const int32_t J = static_cast<int32_t>(drug_ids.size());
    if (J < 1) input_error("build_dataset: need at least one drug");
    const size_t nrec = rec_start.size() - 1;
    auto era_drugs = [&](const std::pair<unsigned, uint32_t>& lo, std::vector<int32_t>& out) {
        const Chunk& ch = chunks[lo.first];
        const LineRec& r = ch.recs[lo.second];
        out.clear();
        for (uint32_t k = 0; k < r.nlabels; ++k) {
            const int32_t local = ch.occ[r.first_label + k];
            out.push_back(fixed ? local : remap[lo.first][static_cast<size_t>(local)]);
        }
        std::sort(out.begin(), out.end());
    };
    std::vector<int32_t> offsets{0}, eps, lens, ys;
    std::vector<uint32_t> drug;
    std::vector<int2> rs;
    std::vector<int32_t> ex;
    int64_t rows = 0;
    int32_t nsub = 0;
    for (size_t s = 0; s < nrec; ++s) {
        int64_t events = 0;
        const std::string_view id = chunks[line_order[rec_start[s]].first].recs[line_order[rec_start[s]].second].subject;
        for (int64_t k = rec_start[s]; k < rec_start[s + 1]; ++k) {
            const LineRec& r = chunks[line_order[k].first].recs[line_order[k].second];
            if (r.length <= 0) input_error("subject '" + std::string(id) + "': era length must be positive");
            if (r.events < 0) input_error("subject '" + std::string(id) + "': negative event count");
            events += r.events;
        }
        if (events == 0) continue; // non-case; carries no information about beta
        for (int64_t k = rec_start[s]; k < rec_start[s + 1]; ++k) {
            const LineRec& r = chunks[line_order[k].first].recs[line_order[k].second];
            if (rows >= 0x7fffffff) input_error("build_dataset: era count overflows the row index type");
            const int32_t row = static_cast<int32_t>(rows++);
            lens.push_back(r.length);
            ys.push_back(r.events);
            era_drugs(line_order[k], ex);
            for (int32_t j : ex) {
                drug.push_back(static_cast<uint32_t>(j));
                rs.push_back(make_int2(row, nsub));
            }
        }
        offsets.push_back(static_cast<int32_t>(rows));
        eps.push_back(static_cast<int32_t>(events));
        ++nsub;
    }
    if (nsub == 0) input_error("build_dataset: no subjects with events remain after exclusion");
    bsccs_dataset* ds = dataset_from_row_pairs(nsub, static_cast<int32_t>(rows), J, static_cast<int64_t>(drug.size()),
                                               offsets.data(), eps.data(), lens.data(), ys.data(), drug.data(),
                                               rs.data(), device, ctas_override);
    ds->drug_ids = std::move(drug_ids);
    return ds;
}

} // namespace bsccs_b200
