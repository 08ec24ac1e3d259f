// io.cpp -- file formats of the reference (see include/subsurf_b200/io.hpp).
// The JSON sidecar is read with a small scanner for the four keys the format
// has ({"dims":[...], "spacing":[...], "dtype":"...", "order":"..."}).
#include "subsurf_b200/io.hpp"

#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <sstream>
#include <vector>

namespace subsurf {

namespace {

std::string slurp(const std::string& path, const char* what) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError(std::string("cannot open ") + what + ": " + path);
    std::ostringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

// value text after "key": in a flat JSON object (no nesting beyond arrays)
std::string json_value(const std::string& text, const std::string& key, const std::string& path) {
    const std::string quoted = "\"" + key + "\"";
    const auto k = text.find(quoted);
    if (k == std::string::npos) throw FormatError("bad image header " + path + ": missing key " + key);
    auto p = text.find(':', k + quoted.size());
    if (p == std::string::npos) throw FormatError("bad image header " + path + ": no value for " + key);
    ++p;
    while (p < text.size() && std::isspace((unsigned char)text[p])) ++p;
    if (p >= text.size()) throw FormatError("bad image header " + path);
    if (text[p] == '[') {
        const auto e = text.find(']', p);
        if (e == std::string::npos) throw FormatError("bad image header " + path + ": unterminated array");
        return text.substr(p + 1, e - p - 1);
    }
    if (text[p] == '"') {
        const auto e = text.find('"', p + 1);
        if (e == std::string::npos) throw FormatError("bad image header " + path + ": unterminated string");
        return text.substr(p + 1, e - p - 1);
    }
    throw FormatError("bad image header " + path + ": unexpected value for " + key);
}

std::vector<double> numbers(const std::string& list, const std::string& path) {
    std::vector<double> out;
    std::stringstream ss(list);
    std::string item;
    while (std::getline(ss, item, ',')) {
        try {
            std::size_t used = 0;
            out.push_back(std::stod(item, &used));
        } catch (const std::exception&) {
            throw FormatError("bad image header " + path + ": not a number: " + item);
        }
    }
    return out;
}

}  // namespace

ImageHeader read_image_header(const std::string& path) {
    const std::string text = slurp(path, "image header");
    ImageHeader h;
    const std::vector<double> dims = numbers(json_value(text, "dims", path), path);
    const std::vector<double> sp = numbers(json_value(text, "spacing", path), path);
    if (dims.size() != 4 || sp.size() != 4)
        throw FormatError("image header needs 4 dims and 4 spacings: " + path);
    for (int a = 0; a < 4; ++a) {
        if (dims[a] != std::floor(dims[a])) throw FormatError("non-integer dim in header: " + path);
        h.dims[a] = (int)dims[a];
        h.spacing[a] = sp[a];
    }
    h.dtype = json_value(text, "dtype", path);
    h.order = json_value(text, "order", path);
    if (h.dtype != "f32le") throw FormatError("unsupported dtype \"" + h.dtype + "\"");
    if (h.order != "i-fastest") throw FormatError("unsupported order \"" + h.order + "\"");
    for (int a = 0; a < 4; ++a) {
        if (h.dims[a] < 1) throw FormatError("non-positive dim in header: " + path);
        if (!(h.spacing[a] > 0.0)) throw FormatError("non-positive spacing: " + path);
    }
    return h;
}

void write_image_header(const ImageHeader& h, const std::string& path) {
    std::ofstream out(path);
    if (!out) throw IoError("cannot write image header: " + path);
    out << std::setprecision(17);
    out << "{\n  \"dims\": [" << h.dims[0] << ", " << h.dims[1] << ", " << h.dims[2] << ", " << h.dims[3]
        << "],\n  \"spacing\": [" << h.spacing[0] << ", " << h.spacing[1] << ", " << h.spacing[2] << ", "
        << h.spacing[3] << "],\n  \"dtype\": \"" << h.dtype << "\",\n  \"order\": \"" << h.order << "\"\n}\n";
}

Field4D read_image4d(const std::string& header_path, const std::string& data_path) {
    static_assert(sizeof(float) == 4, "f32le payload");
    const ImageHeader h = read_image_header(header_path);
    const GridSpec spec = h.grid_spec();
    const std::string raw = slurp(data_path, "image data");
    const std::size_t expected = spec.interior_size() * sizeof(float);
    if (raw.size() != expected)
        throw FormatError("image data " + data_path + ": payload is " + std::to_string(raw.size()) +
                          " bytes, header implies " + std::to_string(expected));
    Field4D f(spec, 0.0);
    const char* p = raw.data();
    for (int l = 1; l <= spec.n4; ++l)
        for (int k = 1; k <= spec.n3; ++k)
            for (int j = 1; j <= spec.n2; ++j)
                for (int i = 1; i <= spec.n1; ++i, p += 4) {
                    float v;
                    std::memcpy(&v, p, 4);  // little-endian hosts only (x86-64 / aarch64)
                    if (!std::isfinite(v)) throw NumericalError("non-finite sample in " + data_path);
                    f.at(i, j, k, l) = (double)v;
                }
    return f;
}

void write_image4d(const Field4D& field, const std::string& header_path, const std::string& data_path) {
    const GridSpec& s = field.spec();
    ImageHeader h;
    h.dims = {s.n1, s.n2, s.n3, s.n4};
    h.spacing = {s.h1, s.h2, s.h3, s.h4};
    write_image_header(h, header_path);
    std::vector<float> buf;
    buf.reserve(s.interior_size());
    for (int l = 1; l <= s.n4; ++l)
        for (int k = 1; k <= s.n3; ++k)
            for (int j = 1; j <= s.n2; ++j)
                for (int i = 1; i <= s.n1; ++i) buf.push_back((float)field.at(i, j, k, l));
    std::ofstream out(data_path, std::ios::binary);
    if (!out) throw IoError("cannot write image data: " + data_path);
    out.write(reinterpret_cast<const char*>(buf.data()), (std::streamsize)(buf.size() * sizeof(float)));
    if (!out) throw IoError("short write on " + data_path);
}

CentersTable read_centers(const std::string& path, const GridSpec& spec) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot open centers file: " + path);
    CentersTable t;
    std::string line;
    std::size_t lineno = 0;
    bool first = true;
    while (std::getline(in, line)) {
        ++lineno;
        if (line.empty()) continue;
        if (first && line.compare(0, 5, "frame") == 0) {  // header line
            first = false;
            continue;
        }
        first = false;
        // exactly the reference's grammar (io.cpp:158-163): a value, then each of the four
        // separators must be the character ',' (whitespace before a token is skipped by >>)
        std::istringstream ss(line);
        CenterRow r;
        char sep[4] = {0, 0, 0, 0};
        ss >> r.frame >> sep[0] >> r.x >> sep[1] >> r.y >> sep[2] >> r.z >> sep[3] >> r.radius;
        const bool commas = sep[0] == ',' && sep[1] == ',' && sep[2] == ',' && sep[3] == ',';
        if (!ss || !commas)
            throw FormatError(path + ":" + std::to_string(lineno) + ": expected frame,x,y,z,radius");
        t.rows.push_back(r);
    }
    validate_centers(t, spec);
    return t;
}

void write_trajectories(const TrajectoryFile& t, const std::string& path) {
    std::ofstream out(path);
    if (!out) throw IoError("cannot write trajectories: " + path);
    out << "trajectory_id,frame,x,y,z\n";  // default ostream formatting, like the reference
    for (const TrajectoryPoint& p : t.points)
        out << p.trajectory_id << ',' << p.frame << ',' << p.x << ',' << p.y << ',' << p.z << "\n";
    if (!out) throw IoError("short write on " + path);
}

TrajectoryFile read_trajectories(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw IoError("cannot open trajectories: " + path);
    TrajectoryFile t;
    std::string line;
    std::size_t lineno = 0;
    while (std::getline(in, line)) {
        ++lineno;
        if (line.empty() || line.compare(0, 13, "trajectory_id") == 0) continue;
        for (char& c : line)
            if (c == ',') c = ' ';
        std::istringstream ss(line);
        TrajectoryPoint p;
        if (!(ss >> p.trajectory_id >> p.frame >> p.x >> p.y >> p.z))
            throw FormatError(path + ":" + std::to_string(lineno) + ": bad trajectory row");
        t.points.push_back(p);
    }
    return t;
}

void export_frame_vtk(const Field4D& field, int l, const std::string& path) {
    const GridSpec& s = field.spec();
    if (l < 1 || l > s.n4)
        throw std::out_of_range("export_frame_vtk: frame " + std::to_string(l) + " outside [1," +
                                std::to_string(s.n4) + "]");
    std::ofstream out(path);
    if (!out) throw IoError("cannot write VTK file: " + path);
    out << "# vtk DataFile Version 3.0\nframe " << l << "\nASCII\nDATASET STRUCTURED_POINTS\n"
        << "DIMENSIONS " << s.n1 << ' ' << s.n2 << ' ' << s.n3 << "\nORIGIN 0 0 0\n"
        << "SPACING " << s.h1 << ' ' << s.h2 << ' ' << s.h3 << "\nPOINT_DATA " << s.frame_interior_size()
        << "\nSCALARS u float 1\nLOOKUP_TABLE default\n";
    for (int k = 1; k <= s.n3; ++k)
        for (int j = 1; j <= s.n2; ++j)
            for (int i = 1; i <= s.n1; ++i) out << (float)field.at(i, j, k, l) << (i == s.n1 ? '\n' : ' ');
    if (!out) throw IoError("short write on " + path);
}

}  // namespace subsurf
